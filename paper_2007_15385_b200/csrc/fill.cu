// fill.cu -- counter-based device point generator (workload input, untimed).
//
// Point j = (min_x + w * U(mix_seed(seed, 2j)), min_y + h * U(mix_seed(seed, 2j+1)))
// with the reference's splitmix64 finaliser (sampling.cpp:107-112) and
// top-53-bit uniform (sampling.cpp:31-33). The affine map is evaluated with
// explicitly rounded f64 operations so the host restatement
// (oracle vo_counter_points_f32) produces the same values bit for bit; the
// f32 variant then rounds once. Stateless per index, so any shard of a
// 2^31-point stream is generated independently on its own GPU.
#include <cstdint>

#include "exact_geom.cuh"
#include "vpipg_internal.h"

namespace vpipg {

namespace {

__device__ __forceinline__ double unit(uint64_t r) {
  return __dmul_rn(static_cast<double>(r >> 11), 0x1.0p-53);
}

template <typename T>
__global__ void fill_kernel(uint64_t seed, uint64_t first, uint64_t m, double min_x, double min_y,
                            double w, double h, T* xs, T* ys) {
  for (uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; t < m;
       t += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t j = first + t;
    xs[t] = static_cast<T>(__dadd_rn(min_x, __dmul_rn(w, unit(mix_seed(seed, 2 * j)))));
    ys[t] = static_cast<T>(__dadd_rn(min_y, __dmul_rn(h, unit(mix_seed(seed, 2 * j + 1)))));
  }
}

}  // namespace

cudaError_t launch_fill_uniform(uint64_t seed, uint64_t first, uint64_t m, double min_x,
                                double min_y, double max_x, double max_y, int dtype, void* xs,
                                void* ys, cudaStream_t stream) {
  if (m == 0) return cudaSuccess;
  const double w = max_x - min_x, h = max_y - min_y;
  const uint64_t blocks64 = (m + 255) / 256;
  const int blocks = static_cast<int>(blocks64 < 148 * 64 ? blocks64 : 148 * 64);
  if (dtype == 0) {
    fill_kernel<double><<<blocks, 256, 0, stream>>>(seed, first, m, min_x, min_y, w, h,
                                                    static_cast<double*>(xs),
                                                    static_cast<double*>(ys));
  } else {
    fill_kernel<float><<<blocks, 256, 0, stream>>>(seed, first, m, min_x, min_y, w, h,
                                                   static_cast<float*>(xs),
                                                   static_cast<float*>(ys));
  }
  return cudaGetLastError();
}

}  // namespace vpipg
