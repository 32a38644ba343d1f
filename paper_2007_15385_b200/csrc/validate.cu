// validate.cu -- device-side engine cross-validation.
//
// Replaces run_validation (bench.cpp:279-308): all three engines on one
// batch, pairwise mask disagreements counted, and every disagreeing point's
// distance to the nearest edge supporting line (edge_line_distance,
// voronoi.cpp:73-82) compared with the band. Works on the ballot words, so a
// 2^31-point batch is cross-checked without a host round trip: one thread per
// mask word XORs the words and only the (rare) disagreeing points touch their
// coordinates. The same kernel compares any two masks of one batch (e.g. the
// reference-exact f64 engine against the fp32 engine) with a relative band.
#include <cstdint>

#include "vpipg_device.cuh"
#include "vpipg_internal.h"

namespace vpipg {

namespace {

__global__ void classify_kernel(const ClassifyArgs a) {
  const uint64_t nwords = (a.m + 31) >> 5;
  unsigned long long pair[3] = {0, 0, 0}, dis = 0, out = 0;
  for (uint64_t w = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; w < nwords;
       w += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t valid = (w + 1 < nwords || (a.m & 31) == 0) ? 0xffffffffu
                                                                 : ((1u << (a.m & 31)) - 1u);
    const uint32_t v = a.w[0][w] & valid, s = a.w[1][w] & valid;
    const uint32_t c = a.w[2] ? (a.w[2][w] & valid) : s;
    pair[0] += __popc(v ^ s);
    pair[1] += __popc(v ^ c);
    pair[2] += __popc(s ^ c);
    uint32_t any = (v ^ s) | (v ^ c);
    dis += __popc(any);
    while (any) {
      const int b = __ffs(any) - 1;
      any &= any - 1;
      const uint64_t j = w * 32 + b;
      double x, y;
      if (a.dtype == 0) {
        x = static_cast<const double*>(a.xs)[j];
        y = static_cast<const double*>(a.ys)[j];
      } else {
        x = static_cast<const float*>(a.xs)[j];
        y = static_cast<const float*>(a.ys)[j];
      }
      double d = INFINITY;
      for (uint32_t k = 0; k < a.n; ++k) {
        const double4 L = a.lines[k];
        d = fmin(d, fabs(L.x * x + L.y * y + L.z));
      }
      double thr = a.band;
      if (a.relative) thr *= fmax(fmax(1.0, a.extent), fmax(fabs(x), fabs(y)));
      const bool outside = d > thr;
      out += outside;
      const unsigned long long slot = atomicAdd(&a.rep->n_recorded, 1ull);
      if (slot < kSampleCapacity) {
        a.rep->sample_index[slot] = j;
        a.rep->sample_dist[slot] = d;
        a.rep->sample_bits[slot] = ((v >> b) & 1u) | (((s >> b) & 1u) << 1) | (((c >> b) & 1u) << 2) |
                                   (outside ? 8u : 0u);
      }
    }
  }
  // warp-reduce then one atomic per warp per counter
#pragma unroll
  for (int sh = 16; sh > 0; sh >>= 1) {
    for (int i = 0; i < 3; ++i) pair[i] += __shfl_xor_sync(0xffffffffu, pair[i], sh);
    dis += __shfl_xor_sync(0xffffffffu, dis, sh);
    out += __shfl_xor_sync(0xffffffffu, out, sh);
  }
  if ((threadIdx.x & 31) == 0) {
    for (int i = 0; i < 3; ++i)
      if (pair[i]) atomicAdd(&a.rep->pair[i], pair[i]);
    if (dis) atomicAdd(&a.rep->disagreeing, dis);
    if (out) atomicAdd(&a.rep->outside_band, out);
  }
}

}  // namespace

cudaError_t launch_classify(const ClassifyArgs& a, cudaStream_t stream) {
  if (a.m == 0) return cudaSuccess;
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const uint64_t nwords = (a.m + 31) >> 5;
  const uint64_t blocks = (nwords + 255) / 256;
  const uint64_t cap = (uint64_t)sms * 8;
  classify_kernel<<<(int)(blocks < cap ? blocks : cap), 256, 0, stream>>>(a);
  return cudaGetLastError();
}

}  // namespace vpipg
