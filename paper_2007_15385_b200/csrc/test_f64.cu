// test_f64.cu -- fp64 batched point-inclusion kernels that repeat the
// reference's arithmetic operation for operation.
//
// The reference is compiled with -ffp-contract=off (proj/CMakeLists.txt:16),
// so each of its expressions is a sequence of individually rounded IEEE
// operations. These kernels issue the same sequence with __dsub_rn /
// __dmul_rn / __dadd_rn (never fused), so every mask byte equals the
// reference's for every input, boundary points included:
//   voronoi_kernel (engines.cpp:65-104): inner_sq <= outer_sq for all k
//   offset_kernel  (engines.cpp:136-160): flags in {0, n}
//   ray_kernel     (engines.cpp:165-204): parity | on-segment latch
// Same warp-tile / ballot / fused-count structure as test_f32.cu.
#include <cstdint>
#include <type_traits>

#include "vpipg_device.cuh"
#include "vpipg_internal.h"

namespace vpipg {

namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
#ifndef VPIPG_F64_P
#define VPIPG_F64_P 8  // points per lane (C5 in f64: 8 -> 83.1 ms, 4 -> 84.9, 2 -> 94.7; C1 equal)
#endif

__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }

// The offset engine's per-point step as explicit PTX, so the comparison
// feeds a predicated increment (one ALU op) instead of an add and a select
// (per-engine kernel at C5 in f64: 21.9 -> 20.1 ms).
// The arithmetic is the reference's, individually rounded.
//
// offset (engines.cpp:150-153): flags += (qy*dvx - qx*dvy < rhs)
__device__ __forceinline__ void offset_step(double x, double y, double dvx, double dvy, double rhs,
                                            uint32_t& flags) {
  asm("{\n\t.reg .pred c;\n\t.reg .f64 t0, t1;\n\t"
      "mul.rn.f64 t0, %2, %3;\n\t"
      "mul.rn.f64 t1, %1, %4;\n\t"
      "sub.rn.f64 t0, t0, t1;\n\t"
      "setp.lt.f64 c, t0, %5;\n\t"
      "@c add.u32 %0, %0, 1;\n\t}"
      : "+r"(flags)
      : "d"(x), "d"(y), "d"(dvx), "d"(dvy), "d"(rhs));
}

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
  if (lane < P && w0 + lane < nwords && a.words) a.words[w0 + lane] = mine;
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

// One engine's test of P points per lane against its per-edge records
// (`tab`: shared or global memory), exactly as the reference computes it.
template <int kEngine, int P>
__device__ __forceinline__ void exact_eval(uint32_t n, double inner_x, double inner_y,
                                           const void* tab, const double (&x)[P],
                                           const double (&y)[P], bool (&in)[P]) {
  if (kEngine == 0) {
    const double2* s = static_cast<const double2*>(tab);
    double inner_sq[P];
#pragma unroll
    for (int p = 0; p < P; ++p) {
      const double dx = dsub(x[p], inner_x), dy = dsub(y[p], inner_y);
      inner_sq[p] = dadd(dmul(dx, dx), dmul(dy, dy));
      in[p] = true;
    }
    for (uint32_t k = 0; k < n; ++k) {
      const double2 g = s[k];
#pragma unroll
      for (int p = 0; p < P; ++p) {
        const double dx = dsub(x[p], g.x), dy = dsub(y[p], g.y);
        const double outer_sq = dadd(dmul(dx, dx), dmul(dy, dy));
        in[p] &= inner_sq[p] <= outer_sq;
      }
    }
  } else if (kEngine == 1) {
    const OffsetEdgeF64* s = static_cast<const OffsetEdgeF64*>(tab);
    uint32_t flags[P];
#pragma unroll
    for (int p = 0; p < P; ++p) flags[p] = 0;
    for (uint32_t e = 0; e < n; ++e) {
      const OffsetEdgeF64 r = s[e];
#pragma unroll
      for (int p = 0; p < P; ++p) {
        offset_step(x[p], y[p], r.dvx, r.dvy, r.rhs, flags[p]);
      }
    }
#pragma unroll
    for (int p = 0; p < P; ++p) in[p] = (flags[p] == 0u) | (flags[p] == n);
  } else {
    // The reference's comparisons with the same operands (ray_kernel), laid
    // out so every per-point boolean is a short-lived predicate (P = 4 or 8
    // points would otherwise carry more predicates than the SM has, and the
    // compiler round-trips them through registers: ~9 SEL / ISETP / LOP3 per
    // point-edge):
    //  - (u.y > qy) and (w.y > qy) both evaluated per edge, as the reference
    //    does, instead of carrying the vertex's bit from the previous edge;
    //  - on_left = (lhs != rhs) & ((lhs > rhs) == going_up) is `lhs > rhs`
    //    for an upward edge and `!(lhs >= rhs)` for a downward one (NaN
    //    included); going_up is uniform, so one comparison per point;
    //  - lhs == rhs only feeds a warp-wide flag; the on-segment box runs (with
    //    lhs recomputed) only when some point of the warp lies exactly on the
    //    edge line, i.e. almost never;
    //  - the parity is an integer toggled under the crossing predicate.
    const RayEdgeF64* s = static_cast<const RayEdgeF64*>(tab);
    uint32_t parity[P], on_edge[P];
#pragma unroll
    for (int p = 0; p < P; ++p) {
      parity[p] = 0;
      on_edge[p] = 0;
    }
    for (uint32_t e = 0; e < n; ++e) {
      const RayEdgeF64 r = s[e];
      bool any_eq = false;
      auto edge = [&](auto up) {
#pragma unroll
        for (int p = 0; p < P; ++p) {
          const bool in_range = (r.uy > y[p]) != (r.wy > y[p]);
          const double lhs = dsub(dmul(y[p], r.dvx), dmul(x[p], r.dvy));
          const bool on_left = decltype(up)::value ? lhs > r.rhs : !(lhs >= r.rhs);
          any_eq |= lhs == r.rhs;
          if (in_range & on_left) parity[p] ^= 1u;
        }
      };
      if (r.going_up) edge(std::true_type{});
      else edge(std::false_type{});
      if (__builtin_expect(__any_sync(0xffffffffu, any_eq), 0)) {
#pragma unroll
        for (int p = 0; p < P; ++p) {
          const double lhs = dsub(dmul(y[p], r.dvx), dmul(x[p], r.dvy));
          on_edge[p] |= (lhs == r.rhs) & (x[p] >= r.min_x) & (x[p] <= r.max_x) &
                        (y[p] >= r.min_y) & (y[p] <= r.max_y);
        }
      }
    }
#pragma unroll
    for (int p = 0; p < P; ++p) in[p] = (on_edge[p] | parity[p]) != 0u;
  }
}

template <int P>
__device__ __forceinline__ void load_tile(const TestArgs& a, uint64_t base, int lane, double (&x)[P],
                                          double (&y)[P]) {
  const double* xs = static_cast<const double*>(a.xs);
  const double* ys = static_cast<const double*>(a.ys);
#pragma unroll
  for (int p = 0; p < P; ++p) {
    const uint64_t idx = base + 32u * p + lane;
    const bool ok = idx < a.m;
    x[p] = ok ? __ldcs(xs + idx) : 0.0;
    y[p] = ok ? __ldcs(ys + idx) : 0.0;
  }
}

// kSmem: per-edge records staged in shared memory (small polygons) or read
// straight from global memory with warp-uniform addresses (any n).
template <int kEngine, int P, bool kSmem>
__global__ void __launch_bounds__(kThreads) exact_kernel(const DevTables t, const TestArgs a) {
  extern __shared__ double4 s_dyn[];
  const uint32_t n = t.n;
  const void* s_tab;
  if (kEngine == 0) {
    double2* s = reinterpret_cast<double2*>(s_dyn);
    if (kSmem)
      for (uint32_t i = threadIdx.x; i < n; i += kThreads) s[i] = t.outer[i];
    s_tab = kSmem ? static_cast<const void*>(s) : t.outer;
  } else if (kEngine == 1) {
    OffsetEdgeF64* s = reinterpret_cast<OffsetEdgeF64*>(s_dyn);
    if (kSmem)
      for (uint32_t i = threadIdx.x; i < n; i += kThreads) s[i] = t.off[i];
    s_tab = kSmem ? static_cast<const void*>(s) : t.off;
  } else {
    RayEdgeF64* s = reinterpret_cast<RayEdgeF64*>(s_dyn);
    if (kSmem)
      for (uint32_t i = threadIdx.x; i < n; i += kThreads) s[i] = t.ray[i];
    s_tab = kSmem ? static_cast<const void*>(s) : t.ray;
  }
  if (kSmem) __syncthreads();
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const uint64_t tiles = (a.m + 32u * P - 1) / (32u * P);
  uint32_t count = 0;
  for (uint64_t tile = (uint64_t)blockIdx.x * kWarps + warp; tile < tiles;
       tile += (uint64_t)gridDim.x * kWarps) {
    const uint64_t base = tile * 32u * P;
    double x[P], y[P];
    bool in[P];
    load_tile<P>(a, base, lane, x, y);
    exact_eval<kEngine, P>(n, t.inner_x, t.inner_y, s_tab, x, y, in);
#pragma unroll
    for (int p = 0; p < P; ++p) in[p] = in[p] & (base + 32u * p + lane < a.m);
    count += emit_words<P>(in, base, a.m, a, lane);
  }
  flush_count(count, a);
}

// All three engines per point in one pass: the points are read once, the
// three record tables sit side by side in shared memory (or stay global).
template <int P, bool kSmem>
__global__ void __launch_bounds__(kThreads) exact_all_kernel(const DevTables t, const TestArgs av,
                                                             const TestArgs ao, const TestArgs ac) {
  extern __shared__ double4 s_dyn[];
  const uint32_t n = t.n;
  double2* sv = reinterpret_cast<double2*>(s_dyn);
  OffsetEdgeF64* so = reinterpret_cast<OffsetEdgeF64*>(sv + n + (n & 1));  // 32-byte aligned
  RayEdgeF64* sr = reinterpret_cast<RayEdgeF64*>(so + n);
  if (kSmem) {
    for (uint32_t i = threadIdx.x; i < n; i += kThreads) {
      sv[i] = t.outer[i];
      so[i] = t.off[i];
      sr[i] = t.ray[i];
    }
    __syncthreads();
  }
  const void* tv = kSmem ? static_cast<const void*>(sv) : t.outer;
  const void* to = kSmem ? static_cast<const void*>(so) : t.off;
  const void* tr = kSmem ? static_cast<const void*>(sr) : t.ray;
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const uint64_t tiles = (av.m + 32u * P - 1) / (32u * P);
  uint32_t cv = 0, co = 0, cc = 0;
  for (uint64_t tile = (uint64_t)blockIdx.x * kWarps + warp; tile < tiles;
       tile += (uint64_t)gridDim.x * kWarps) {
    const uint64_t base = tile * 32u * P;
    double x[P], y[P];
    bool in[P];
    load_tile<P>(av, base, lane, x, y);
    exact_eval<0, P>(n, t.inner_x, t.inner_y, tv, x, y, in);
#pragma unroll
    for (int p = 0; p < P; ++p) in[p] = in[p] & (base + 32u * p + lane < av.m);
    cv += emit_words<P>(in, base, av.m, av, lane);
    exact_eval<1, P>(n, t.inner_x, t.inner_y, to, x, y, in);
#pragma unroll
    for (int p = 0; p < P; ++p) in[p] = in[p] & (base + 32u * p + lane < ao.m);
    co += emit_words<P>(in, base, ao.m, ao, lane);
    exact_eval<2, P>(n, t.inner_x, t.inner_y, tr, x, y, in);
#pragma unroll
    for (int p = 0; p < P; ++p) in[p] = in[p] & (base + 32u * p + lane < ac.m);
    cc += emit_words<P>(in, base, ac.m, ac, lane);
  }
  flush_count(cv, av);
  flush_count(co, ao);
  flush_count(cc, ac);
}

template <int kEngine>
cudaError_t launch_one(const DevTables& t, const TestArgs& a, size_t rec_bytes,
                       cudaStream_t stream) {
  constexpr int P = VPIPG_F64_P;
  const bool staged = (size_t)t.n * rec_bytes <= 96 * 1024;
  auto k = staged ? exact_kernel<kEngine, P, true> : exact_kernel<kEngine, P, false>;
  const size_t smem = staged ? (size_t)t.n * rec_bytes : 0;
  int sms = 0, per_sm = 0;
  cudaError_t e = launch_config(reinterpret_cast<const void*>(k), kThreads, smem, &sms, &per_sm);
  if (e != cudaSuccess) return e;
  const uint64_t need = (a.m + kThreads * P - 1) / (kThreads * P);
  const uint64_t cap = (uint64_t)sms * per_sm;
  const int grid = static_cast<int>(need < cap ? (need ? need : 1) : cap);
  k<<<grid, kThreads, smem, stream>>>(t, a);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_test_f64_all(const DevTables& t, const TestArgs* a, cudaStream_t stream) {
  constexpr int P = VPIPG_F64_P;
  const size_t rec = sizeof(double2) + sizeof(OffsetEdgeF64) + sizeof(RayEdgeF64);
  const size_t bytes = (size_t)t.n * rec + sizeof(double2);
  const bool staged = bytes <= 96 * 1024;
  auto k = staged ? exact_all_kernel<P, true> : exact_all_kernel<P, false>;
  const size_t smem = staged ? bytes : 0;
  int sms = 0, per_sm = 0;
  cudaError_t e = launch_config(reinterpret_cast<const void*>(k), kThreads, smem, &sms, &per_sm);
  if (e != cudaSuccess) return e;
  const uint64_t need = (a[0].m + kThreads * P - 1) / (kThreads * P);
  const uint64_t cap = (uint64_t)sms * per_sm;
  const int grid = static_cast<int>(need < cap ? (need ? need : 1) : cap);
  k<<<grid, kThreads, smem, stream>>>(t, a[0], a[1], a[2]);
  return cudaGetLastError();
}

cudaError_t launch_test_f64(const DevTables& t, int engine, const TestArgs& a,
                            cudaStream_t stream) {
  switch (engine) {
    case 0: return launch_one<0>(t, a, sizeof(double2), stream);
    case 1: return launch_one<1>(t, a, sizeof(OffsetEdgeF64), stream);
    default: return launch_one<2>(t, a, sizeof(RayEdgeF64), stream);
  }
}

}  // namespace vpipg
