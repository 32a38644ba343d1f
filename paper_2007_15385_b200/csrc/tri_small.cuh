// tri_small.cuh -- the small-polygon fused three-engine kernel (fp32):
// templates shared by tri_small.cu (3..8 vertices, the route's plan and entry
// points) and tri_small_hi.cu (9..12 vertices), two translation units so the
// instantiations compile in parallel.
//
// vpipg_test_multi with all three engines on a polygon of at most kSmallMaxN
// crossing vertices whose Voronoi and sign-of-offset slab tables share one
// single-section form: voronoi_kernel (engines.cpp:65-104), offset_kernel
// (engines.cpp:136-160) and ray_kernel (engines.cpp:165-204) over one read of
// the points, as tri_kernel (test_f32.cu) does for any n, but with the edge
// count and the slab group size as template parameters.
#pragma once

#include <cstdint>
#include <cstring>
#include <type_traits>

#include "f32_common.cuh"
#include "vpipg_internal.h"

namespace vpipg {

namespace {


// ---------------------------------------------------------------------------
// Small-polygon fused pass (tri_small_kernel): the three engines for polygons
// of at most kSmallMaxN crossing vertices whose two slab tables share one
// single-section form (y-only or x-only). The vertex count NC and the padded
// record count K of the slab groups are compile-time, so every table value is
// a constant-bank operand of its FFMA / FADD (no table loads, no edge loops,
// no group-count branches) and each point runs straight-line code, point
// after point. The arithmetic is the per-engine kernels' own: the crossing
// pairs edges (0,1), (2,3), ... with the same anchoring (CrossEngine), and
// a slab group padded with copies of its first record takes the same max /
// min (both are exact and idempotent), so the masks equal the generic fused
// kernel's bit for bit. At n = 3 the generic kernel issues 50.6 instructions
// per point for the three engines, ~13 of them loop and group bookkeeping
// (profiles/ncu_full_r02_c3n3.json).
#ifndef VPIPG_TRI_SMALL_P
#define VPIPG_TRI_SMALL_P 16
#endif
#ifndef VPIPG_TRI_SMALL
#define VPIPG_TRI_SMALL 1
#endif
// points per lane per slice: 16 up to 8 vertices; 12 above (C2, n = 12 and
// 2^24 points: 74 us against 77 at P = 16 and 76 at P = 8, whose unrolled
// slices also stall less on instruction fetch; at 2^28 points P = 16 is
// ~1 % faster for 10-12 vertices)
#ifndef VPIPG_TRI_SMALL_P_HI
#define VPIPG_TRI_SMALL_P_HI 12
#endif
constexpr int small_p(int nc) { return nc <= 8 ? VPIPG_TRI_SMALL_P : VPIPG_TRI_SMALL_P_HI; }
constexpr int kSmallMaxN = 12;
// padded slab group sizes K (records of two lines) instantiated per vertex
// count: a single-section group of a convex NC-gon holds at most NC - 1
// lines (the other side holds at least one), i.e. up to NC / 2 records, and
// the fuller side at least ceil(NC / 2) lines, i.e. at least ceil(NC / 4)
// records -- every K in between is instantiated (above 8 vertices from that
// lower bound up: groups that hold fewer lines are padded to it)
constexpr int small_kmin(int nc) { return nc <= 8 ? 1 : (nc + 3) / 4; }
constexpr int small_kmax(int nc) { return nc / 2; }

template <int NC, int K>
struct TriSmallParams {
  float ox, oy;          // local frame of the slab tables (0, 0: absolute)
  float4 slab[2][2][K];  // [Voronoi | offset][lo | hi][record]: (B0, C0, B1, C1)
  float4 cross[NC];      // crossing records in the absolute frame
};

// crossing parity word of one point (CrossEngine::eval, unrolled)
template <int NC>
__device__ __forceinline__ uint32_t cross_one(const float4 (&c)[NC], float x, float y) {
  uint32_t par = 0;
  float hp = y - c[NC - 1].y;
#pragma unroll
  for (int k = 0; k + 1 < NC; k += 2) {
    const float h0 = y - c[k].y, g0 = c[k].x - x;
    const float h1 = y - c[k + 1].y;
    par ^= cross_bit(h0, hp, fmaf(h0, c[k].z, g0)) ^ cross_bit(h1, h0, fmaf(h0, c[k + 1].z, g0));
    hp = h1;
  }
  if constexpr (NC & 1) {
    const float h0 = y - c[NC - 1].y;
    par ^= cross_bit(h0, hp, fmaf(h0, c[NC - 1].z, c[NC - 1].x - x));
  }
  return par;
}

// one single-section slab test (SlabEngine::section): MODE 1 bounds y by
// lines in x, MODE 2 bounds x by lines in y; inside iff hi >= lo
template <int K, int MODE>
__device__ __forceinline__ void slab_one(const float4 (&t)[2][K], float x, float y, float& lo,
                                         float& hi) {
  const float v = MODE == 1 ? x : y, w = MODE == 1 ? y : x;
  lo = w;
  hi = w;
#pragma unroll
  for (int i = 0; i < K; ++i) {
    const float4 a = t[0][i], b = t[1][i];
    lo = fmax3(lo, fmaf(a.x, v, a.y), fmaf(a.z, v, a.w));
    hi = fmin3(hi, fmaf(b.x, v, b.y), fmaf(b.z, v, b.w));
  }
}

// votes, counts and stores of one engine over a slice, four words at a time
// (f(p, a, b) gives point p's vote operands; see emit). Full slices store
// their words with predicated 16-byte stores and no byte masks (small_plan
// takes only 16-byte aligned word outputs and no byte outputs); the guarded
// tail keeps emit's general stores.
template <bool kGuard, int kVote, int P, class F>
__device__ __forceinline__ cnt_t emit4(F&& f, uint64_t base, const TestArgs& a, int lane, bool live) {
  static_assert(P % 4 == 0, "16-byte word stores need P % 4 == 0");
  cnt_t cnt = 0;
  const uint64_t w0 = base >> 5;
  const bool st = live && lane == 0 && a.words != nullptr;
#pragma unroll
  for (int q = 0; q < P / 4; ++q) {
    uint32_t w[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int p = 4 * q + j;
      float va, vb;
      f(p, va, vb);
      if (kGuard && base + 32u * p + lane >= a.m) va = kVote == 2 ? 0.f : -INFINITY;
      w[j] = vote_in<kVote>(va, vb, cnt);
    }
    if constexpr (!kGuard) {
      if (st) __stcs(reinterpret_cast<uint4*>(a.words + w0) + q, make_uint4(w[0], w[1], w[2], w[3]));
    } else {
      const uint64_t nwords = (a.m + 31) >> 5;
      if (st) {
#pragma unroll
        for (int j = 0; j < 4; ++j)
          if (w0 + 4 * q + j < nwords) a.words[w0 + 4 * q + j] = w[j];
      }
      if (live && a.bytes) {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const uint64_t idx = base + 32u * (4 * q + j) + lane;
          if (idx < a.m) a.bytes[idx] = (w[j] >> lane) & 1u;
        }
      }
    }
  }
  return live ? cnt : 0;
}

template <int NC, int K, int MODE, bool kGuard, bool kShift>
__device__ __forceinline__ void tri_small_slice(const TriSmallParams<NC, K>& prm, const TestArgs& av,
                                                const TestArgs& ao, const TestArgs& ac,
                                                uint64_t base, int lane, bool live, cnt_t& cv,
                                                cnt_t& co, cnt_t& cc) {
  constexpr int P = small_p(NC);
  const float* xs = static_cast<const float*>(av.xs) + base + lane;
  const float* ys = static_cast<const float*>(av.ys) + base + lane;
  float x[P], y[P];
#pragma unroll
  for (int p = 0; p < P; ++p) {
    const bool ok = !kGuard || base + 32u * p + lane < av.m;
    x[p] = ok ? __ldcs(xs + 32 * p) : 0.f;
    y[p] = ok ? __ldcs(ys + 32 * p) : 0.f;
  }
  // crossing on the points as loaded (absolute-frame table), as tri_kernel;
  // for 5-8 vertices (and no local-frame shift, which must follow it) after
  // the two slab engines, which measured faster there (C3 n = 8: 0.735 ->
  // 0.710 ms; n = 5-7 1-3 %); first below (n = 3-4: 5-6 % slower last) and
  // above (C2, n = 12: 1 % slower last)
  auto crossing = [&] {
    cc += emit4<kGuard, 2, P>(
        [&](int p, float& a, float& b) {
          a = __uint_as_float(cross_one<NC>(prm.cross, x[p], y[p]));
          b = 0.f;
        },
        base, ac, lane, live);
  };
  constexpr bool kCrossLast = !kShift && NC >= 5 && NC <= 8;
  if constexpr (!kCrossLast) crossing();
  if constexpr (kShift) {
#pragma unroll
    for (int p = 0; p < P; ++p) {
      x[p] -= prm.ox;
      y[p] -= prm.oy;
    }
  }
  cv += emit4<kGuard, 0, P>([&](int p, float& a, float& b) { slab_one<K, MODE>(prm.slab[0], x[p], y[p], b, a); },
                            base, av, lane, live);
  co += emit4<kGuard, 1, P>([&](int p, float& a, float& b) { slab_one<K, MODE>(prm.slab[1], x[p], y[p], b, a); },
                            base, ao, lane, live);
  if constexpr (kCrossLast) crossing();
}

#ifndef VPIPG_TRI_SMALL_MINB
#define VPIPG_TRI_SMALL_MINB 2
#endif
template <int NC, int K, int MODE>
__global__ void __launch_bounds__(kThreads, VPIPG_TRI_SMALL_MINB)
    tri_small_kernel(const __grid_constant__ TriSmallParams<NC, K> prm, const TestArgs av,
                     const TestArgs ao, const TestArgs ac, const uint64_t full_slices) {
  constexpr int P = small_p(NC);
  constexpr int kWarpPts = 32 * P;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const SliceRounds sr(full_slices, warp);
  const float* xs = static_cast<const float*>(av.xs);
  const float* ys = static_cast<const float*>(av.ys);
  constexpr int kLines = kWarpPts * 4 / 128;
  auto prefetch = [&](uint64_t r) {
    if (r >= sr.rounds) return;
    const uint64_t g = sr.slice(r);
    for (int l = lane; l < 2 * kLines; l += 32)
      prefetch_l2((l < kLines ? xs : ys) + g * kWarpPts + (l % kLines) * 32);
  };
  cnt_t cv = 0, co = 0, cc = 0;
  // the slab engines' local-frame shift only where prep moved the origin
  // (to_local's test, hoisted out of the slice loop)
  auto run = [&](auto shift) {
    constexpr bool S = decltype(shift)::value;
    prefetch(0);
    for (uint64_t r = 0; r < sr.rounds; ++r) {
      prefetch(r + 1);
      tri_small_slice<NC, K, MODE, false, S>(prm, av, ao, ac, sr.slice(r) * kWarpPts, lane,
                                             sr.live(r), cv, co, cc);
    }
    if (sr.g0 == full_slices % sr.W) {
      for (uint64_t base = full_slices * kWarpPts; base < av.m; base += kWarpPts)
        tri_small_slice<NC, K, MODE, true, S>(prm, av, ao, ac, base, lane, true, cv, co, cc);
    }
  };
  if (prm.ox != 0.f || prm.oy != 0.f) run(std::true_type{});
  else run(std::false_type{});
  flush_count(cv, av);
  flush_count(co, ao);
  flush_count(cc, ac);
}

template <int NC, int K, int MODE>
cudaError_t launch_small(const DevTables& t, const TestArgs* a, cudaStream_t stream) {
  constexpr int kWarpPts = 32 * small_p(NC);
  TriSmallParams<NC, K> prm{};
  prm.ox = t.ox;
  prm.oy = t.oy;
  const int glo = MODE == 1 ? kGroupYlo : kGroupXlo;
  for (int e = 0; e < 2; ++e)
    for (int s = 0; s < 2; ++s) {
      const float2* g = t.h_slab[e] + t.slab[e].off[glo + s];
      const uint32_t c = t.slab[e].cnt[glo + s] / 2;
      for (int i = 0; i < K; ++i)  // padded with copies of the first record
        std::memcpy(&prm.slab[e][s][i], g + 2 * (i < (int)c ? i : 0), sizeof(float4));
    }
  for (int k = 0; k < NC; ++k) prm.cross[k] = cross_record_abs(t.h_cross[k], t.ox, t.oy);
  auto kern = tri_small_kernel<NC, K, MODE>;
  int sms = 0, per_sm = 0;
  cudaError_t e = launch_config(reinterpret_cast<const void*>(kern), kThreads, 0, &sms, &per_sm);
  if (e != cudaSuccess) return e;
  const uint64_t full_slices = a[0].m / kWarpPts;
  const uint64_t cap = (uint64_t)sms * per_sm;
  const uint64_t want = (full_slices + kWarps - 1) / kWarps;
  kern<<<(int)(want < cap ? want : cap), kThreads, 0, stream>>>(prm, a[0], a[1], a[2], full_slices);
  return cudaGetLastError();
}

// the instantiation for vertex count NC and table form MODE with padded
// group size k, or null
template <int NC, int MODE, int K = small_kmin(NC)>
auto small_for_k(int k) -> cudaError_t (*)(const DevTables&, const TestArgs*, cudaStream_t) {
  if constexpr (K > small_kmax(NC)) return nullptr;
  else return k == K ? launch_small<NC, K, MODE> : small_for_k<NC, MODE, K + 1>(k);
}
}  // namespace

using SmallLaunch = cudaError_t (*)(const DevTables&, const TestArgs*, cudaStream_t);
// the launcher of the instantiation for (vertex count nc, padded group size
// k, table form mode) or null: 3..8 vertices (tri_small.cu), 9..12 (tri_small_hi.cu)
SmallLaunch small_launcher_lo(int nc, int k, int mode);
SmallLaunch small_launcher_hi(int nc, int k, int mode);

}  // namespace vpipg
