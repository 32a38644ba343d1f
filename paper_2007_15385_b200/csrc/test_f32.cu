// test_f32.cu -- fp32 batched point-inclusion kernels for sm_100a.
//
// Replaces the reference's batch kernels for float32 point streams:
//   voronoi_kernel   (engines.cpp:65-104)  -> slab kernel, Voronoi table
//   offset_kernel    (engines.cpp:136-160) -> slab kernel, offset table
//   ray_kernel       (engines.cpp:165-204) -> crossing kernel
//   count_inside     (engines.cpp:215-217) -> fused popc + one atomic per warp
//
// Work decomposition: a warp owns "warp tiles" of 32*P consecutive points;
// lane l handles points base + 32*p + l (p < P), so the ballot of sub-tile p
// is exactly mask word (base/32 + p) in the PIPM bit order (io.cpp:272-279)
// and every global load / store is a fully coalesced 128-byte line per warp.
// The polygon's coefficient table is staged once per CTA in shared memory and
// read with warp-uniform (broadcast) 16-byte loads; every point-edge costs one
// FFMA plus half an FMNMX3 (slab) -- no per-point data-dependent branches,
// like the reference's branch-free kernels.
#include <cstdint>

#include "vpipg_device.cuh"
#include "vpipg_internal.h"

namespace vpipg {

namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;

__device__ __forceinline__ float fmax3(float a, float b, float c) {
  float r;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
  return r;
}
__device__ __forceinline__ float fmin3(float a, float b, float c) {
  float r;
  asm("min.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
  return r;
}

// Streaming loads: every point is read exactly once.
__device__ __forceinline__ float ld_stream(const float* p) { return __ldcs(p); }

// Emits the P ballot words of one warp tile: lane p keeps word p; lanes
// 0..P-1 store them (one coalesced 4P-byte store) and count their bits.
template <int P>
__device__ __forceinline__ uint32_t emit_words(const bool (&in)[P], uint64_t base, uint64_t m,
                                               const TestArgs& a, int lane) {
  uint32_t mine = 0;
#pragma unroll
  for (int p = 0; p < P; ++p) {
    const uint32_t w = __ballot_sync(0xffffffffu, in[p]);
    if (lane == p) mine = w;
  }
  const uint64_t w0 = base >> 5;
  const uint64_t nwords = (m + 31) >> 5;
  if (lane < P && w0 + lane < nwords) {
    if (a.words) __stcs(a.words + w0 + lane, mine);
  }
  if (a.bytes) {
#pragma unroll
    for (int p = 0; p < P; ++p) {
      const uint64_t idx = base + 32u * p + lane;
      if (idx < m) a.bytes[idx] = in[p] ? 1 : 0;
    }
  }
  return lane < P ? __popc(mine) : 0u;
}

__device__ __forceinline__ void flush_count(uint32_t cnt, const TestArgs& a) {
#pragma unroll
  for (int s = 16; s > 0; s >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, s);
  if ((threadIdx.x & 31) == 0 && a.inside && cnt) atomicAdd(a.inside, (unsigned long long)cnt);
}

// ---------------------------------------------------------------------------
// Slab kernel: Voronoi and sign-of-offset (same arithmetic, different table).
template <int P>
__global__ void __launch_bounds__(kThreads) slab_kernel(const SlabTable tab, const float ox,
                                                        const float oy, const TestArgs a) {
  extern __shared__ float4 s_coef4[];  // (B0, C0, B1, C1) pairs of edges
  {
    const float4* src = reinterpret_cast<const float4*>(tab.coef);
    for (uint32_t i = threadIdx.x; i < tab.total / 2; i += kThreads) s_coef4[i] = src[i];
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const float* xs = static_cast<const float*>(a.xs);
  const float* ys = static_cast<const float*>(a.ys);
  const uint64_t tiles = (a.m + 32u * P - 1) / (32u * P);
  const uint32_t g0 = tab.off[0] / 2, n0 = tab.cnt[0] / 2;
  const uint32_t g1 = tab.off[1] / 2, n1 = tab.cnt[1] / 2;
  const uint32_t g2 = tab.off[2] / 2, n2 = tab.cnt[2] / 2;
  const uint32_t g3 = tab.off[3] / 2, n3 = tab.cnt[3] / 2;
  uint32_t count = 0;
  for (uint64_t tile = (uint64_t)blockIdx.x * kWarps + warp; tile < tiles;
       tile += (uint64_t)gridDim.x * kWarps) {
    const uint64_t base = tile * 32u * P;
    float x[P], y[P];
    bool in[P];
#pragma unroll
    for (int p = 0; p < P; ++p) {
      const uint64_t idx = base + 32u * p + lane;
      const bool ok = idx < a.m;
      x[p] = (ok ? ld_stream(xs + idx) : 0.f) - ox;
      y[p] = (ok ? ld_stream(ys + idx) : 0.f) - oy;
    }
    float lo[P], hi[P];
#pragma unroll
    for (int p = 0; p < P; ++p) { lo[p] = -INFINITY; hi[p] = INFINITY; }
    // x' >= B y' + C  (max over XLO), x' <= B y' + C (min over XHI)
    for (uint32_t i = 0; i < n0; ++i) {
      const float4 c = s_coef4[g0 + i];
#pragma unroll
      for (int p = 0; p < P; ++p) lo[p] = fmax3(lo[p], fmaf(c.x, y[p], c.y), fmaf(c.z, y[p], c.w));
    }
    for (uint32_t i = 0; i < n1; ++i) {
      const float4 c = s_coef4[g1 + i];
#pragma unroll
      for (int p = 0; p < P; ++p) hi[p] = fmin3(hi[p], fmaf(c.x, y[p], c.y), fmaf(c.z, y[p], c.w));
    }
#pragma unroll
    for (int p = 0; p < P; ++p) {
      in[p] = (x[p] >= lo[p]) & (x[p] <= hi[p]);
      lo[p] = -INFINITY;
      hi[p] = INFINITY;
    }
    // y' >= B x' + C (max over YLO), y' <= B x' + C (min over YHI)
    for (uint32_t i = 0; i < n2; ++i) {
      const float4 c = s_coef4[g2 + i];
#pragma unroll
      for (int p = 0; p < P; ++p) lo[p] = fmax3(lo[p], fmaf(c.x, x[p], c.y), fmaf(c.z, x[p], c.w));
    }
    for (uint32_t i = 0; i < n3; ++i) {
      const float4 c = s_coef4[g3 + i];
#pragma unroll
      for (int p = 0; p < P; ++p) hi[p] = fmin3(hi[p], fmaf(c.x, x[p], c.y), fmaf(c.z, x[p], c.w));
    }
#pragma unroll
    for (int p = 0; p < P; ++p) {
      const uint64_t idx = base + 32u * p + lane;
      in[p] = in[p] & (y[p] >= lo[p]) & (y[p] <= hi[p]) & (idx < a.m);
    }
    count += emit_words<P>(in, base, a.m, a, lane);
  }
  flush_count(count, a);
}

// ---------------------------------------------------------------------------
// Crossing kernel (engines.cpp:165-204). For edge w = v[k-1] -> u = v[k]:
//   in_range  <=>  (u.y > qy) != (w.y > qy)  <=>  sign(h_k) ^ sign(h_{k-1}),
//                  h = qy - v.y (never -0.0: see prep.cu)
//   on_left   <=>  qx < x-of-edge-at-qy  <=>  d = (w.x - qx) + h_{k-1} * dvx/dvy > 0
// crossing bit = (H_k ^ H_{k-1}) & ~D, parity accumulated by XOR in bit 31.
// Points exactly on an edge line are inside the 1e-5 parity band, so the
// reference's closed-boundary latch (engines.cpp:194-196) is not repeated in
// fp32; the f64 kernel repeats it exactly.
template <int P>
__global__ void __launch_bounds__(kThreads) cross_kernel(const CrossTable tab, const float ox,
                                                         const float oy, const TestArgs a) {
  extern __shared__ float4 s_vert[];
  for (uint32_t i = threadIdx.x; i < tab.n; i += kThreads) s_vert[i] = tab.vert[i];
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const float* xs = static_cast<const float*>(a.xs);
  const float* ys = static_cast<const float*>(a.ys);
  const uint64_t tiles = (a.m + 32u * P - 1) / (32u * P);
  const uint32_t n = tab.n;
  uint32_t count = 0;
  for (uint64_t tile = (uint64_t)blockIdx.x * kWarps + warp; tile < tiles;
       tile += (uint64_t)gridDim.x * kWarps) {
    const uint64_t base = tile * 32u * P;
    float x[P], y[P];
#pragma unroll
    for (int p = 0; p < P; ++p) {
      const uint64_t idx = base + 32u * p + lane;
      const bool ok = idx < a.m;
      x[p] = (ok ? ld_stream(xs + idx) : 0.f) - ox;
      y[p] = (ok ? ld_stream(ys + idx) : 0.f) - oy;
    }
    uint32_t par[P];
    bool in[P];
    if (n > 0) {
      const float4 last = s_vert[n - 1];
      float hp[P], gp[P];
#pragma unroll
      for (int p = 0; p < P; ++p) {
        hp[p] = y[p] - last.y;
        gp[p] = last.x - x[p];
        par[p] = 0;
      }
      for (uint32_t k = 0; k < n; ++k) {
        const float4 v = s_vert[k];
#pragma unroll
        for (int p = 0; p < P; ++p) {
          const float h = y[p] - v.y;
          const float d = fmaf(hp[p], v.z, gp[p]);
          par[p] ^= (__float_as_uint(h) ^ __float_as_uint(hp[p])) & ~__float_as_uint(d);
          hp[p] = h;
          gp[p] = v.x - x[p];
        }
      }
    } else {
#pragma unroll
      for (int p = 0; p < P; ++p) par[p] = 0;
    }
#pragma unroll
    for (int p = 0; p < P; ++p) {
      const uint64_t idx = base + 32u * p + lane;
      in[p] = (par[p] >> 31) & (idx < a.m);
    }
    count += emit_words<P>(in, base, a.m, a, lane);
  }
  flush_count(count, a);
}

template <class K>
int grid_for(K kernel, size_t smem, uint64_t m, int pts_per_block) {
  int dev = 0, sms = 0, per_sm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, kThreads, smem);
  if (per_sm < 1) per_sm = 1;
  const uint64_t need = (m + pts_per_block - 1) / pts_per_block;
  const uint64_t cap = (uint64_t)sms * per_sm;
  return static_cast<int>(need < cap ? (need ? need : 1) : cap);
}

}  // namespace

cudaError_t launch_test_f32(const DevTables& t, int engine, const TestArgs& a,
                            cudaStream_t stream) {
  constexpr int P = 8;
  if (engine == 0 || engine == 1) {
    const SlabTable& tab = t.slab[engine];
    const size_t smem = (size_t)tab.total * sizeof(float2);
    auto k = slab_kernel<P>;
    if (smem > 48 * 1024) {
      cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e != cudaSuccess) return e;
    }
    const int grid = grid_for(k, smem, a.m, kThreads * P);
    k<<<grid, kThreads, smem, stream>>>(tab, t.ox, t.oy, a);
    return cudaGetLastError();
  }
  const size_t smem = (size_t)t.cross.n * sizeof(float4);
  auto k = cross_kernel<P>;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  const int grid = grid_for(k, smem, a.m, kThreads * P);
  k<<<grid, kThreads, smem, stream>>>(t.cross, t.ox, t.oy, a);
  return cudaGetLastError();
}

}  // namespace vpipg
