// test_f32.cu -- fp32 batched point-inclusion kernels for sm_100a.
//
// Replaces the reference's batch kernels for float32 point streams:
//   voronoi_kernel   (engines.cpp:65-104)  -> SlabEngine, Voronoi table
//   offset_kernel    (engines.cpp:136-160) -> SlabEngine, offset table
//   ray_kernel       (engines.cpp:165-204) -> CrossEngine
//   count_inside     (engines.cpp:215-217) -> fused popc + one atomic per warp
//
// Streaming structure: a persistent grid; every warp streams its own slices of
// 32*P points (slice g goes to warp g mod W), two ways, chosen per engine by
// measurement:
//  - stream_kernel (crossing): a private kStages-deep shared-memory ring per
//    warp filled with cp.async.bulk (the 1-D TMA path, evict-first). Lane 0
//    arms the stage's "full" mbarrier with the expected bytes; after the warp
//    copied a stage into registers, all 32 lanes arrive on its "empty"
//    mbarrier (release) and lane 0 refills it with slice g + S*W, so loads run
//    kStages slices ahead of the math with no cross-warp coupling.
//  - ldg_kernel (slab engines): coalesced loads straight into registers after
//    an L2 prefetch of the slice two rounds ahead.
// Lane l owns points 32*p + l (p < P) of a slice, so the ballot of sub-tile p
// is exactly one PIPM mask word (io.cpp:272-279, bit j = point j) and word
// stores are coalesced. The polygon table is staged once per CTA in shared
// memory and read with warp-uniform 16-byte broadcasts. generic_kernel handles
// unaligned inputs with guarded direct loads.
#include <cstdint>
#include <cstring>
#include <type_traits>

#include "f32_common.cuh"
#include "tma_pipe.cuh"
#include "vpipg_device.cuh"
#include "vpipg_internal.h"

// points per lane per slice (tuned on C5, profiles/crossing_forms_r02.json):
// the slab kernel amortises its per-slice work best at 20 (16: +0.6 %), the
// crossing kernel, which carries one h per point, at 20 (12 / 16 / 24:
// +8 / +4 / -1 %; 24 spills with shared-memory tables); all run 2 CTAs of
// 8 warps per SM
#ifndef VPIPG_SLAB_P
#define VPIPG_SLAB_P 20
#endif
#ifndef VPIPG_CROSS_P
#define VPIPG_CROSS_P 20
#endif
#ifndef VPIPG_CROSS_VOTE
#define VPIPG_CROSS_VOTE 2
#endif
#ifndef VPIPG_SLAB_UNROLL
#define VPIPG_SLAB_UNROLL 1
#endif
#ifndef VPIPG_CROSS_UNROLL
#define VPIPG_CROSS_UNROLL 1
#endif

namespace vpipg {

namespace {

constexpr int kStages = 2;            // per-warp ring depth

// ---------------------------------------------------------------------------
#ifndef VPIPG_LOCAL_FRAME
#define VPIPG_LOCAL_FRAME 1
#endif
// Points enter every engine in the polygon-local frame, x' = x - ox, y' = y - oy
// with (ox, oy) = the f32-rounded centroid (prep.cu): exact (Sterbenz) for every
// point within a factor of two of the origin's coordinates, i.e. near a polygon
// far from the origin, so the table arithmetic errs by ~2^-24 of the polygon's
// extent there, not of |x|.
//
// The shift is skipped (a uniform branch) when prep put the origin at (0, 0):
// polygons whose centroid lies within their own extent of the origin, where
// the absolute frame is as accurate (prep.cu).
template <int P>
__device__ __forceinline__ void to_local(float (&x)[P], float (&y)[P], float ox, float oy) {
  if (ox != 0.f || oy != 0.f) {
#pragma unroll
    for (int p = 0; p < P; ++p) {
      x[p] -= ox;
      y[p] -= oy;
    }
  }
}

// Slab engine (Voronoi and sign-of-offset): inside iff
//   max(XLO) <= x' <= min(XHI)  and  max(YLO) <= y' <= min(YHI)
// where each group entry is t = B * (other coordinate) + C (see prep.cu).
// kNanIn: the answer for a point with a NaN coordinate, the reference's
// IEEE behaviour -- Voronoi `inner_sq <= outer_sq` is false (outside),
// sign-of-offset raises no flag, so flags == 0 (inside).
struct SlabParams {
  SlabTable tab;
  float ox, oy;
};

// Tables of up to kInlineMax float4 records can travel in the kernel's
// parameter bank instead of shared memory (VPIPG_INLINE): the edge loops then
// read them with uniform constant loads (LDCU) into uniform registers, so the
// per-edge FFMA / FADD operands come from the uniform datapath and no vector
// register or shared-memory load is spent on table values.
constexpr int kInlineMax = 128;
struct SlabParamsInl {
  SlabTable tab;
  float ox, oy;
  float4 v[kInlineMax];
};

// kMode: 0 = two sections (mixed table), 1 = y-only table, 2 = x-only table
// (prep.cu slab_scatter), -1 = decided per launch from the table counts (the
// fused kernel); the launcher instantiates the mode the table has, so each
// streaming kernel carries one code path
template <int P, bool kNanIn, int kMode = -1, bool kInline = false>
struct SlabEngine {
  static constexpr int kP = P;
  static constexpr int kVote = kNanIn ? 1 : 0;  // see vote_in
  static constexpr bool kRegStream = true;  // ldg_kernel
  static constexpr bool kInl = kInline;
  static constexpr bool kUniform = false;
  static constexpr bool kShiftIn = VPIPG_LOCAL_FRAME;  // points enter in the local frame
  // shared by every (P, NaN rule, form) instantiation of one table placement
  using Params = std::conditional_t<kInline, SlabParamsInl, SlabParams>;
  static size_t table_bytes(const Params& p) { return kInline ? 0 : (size_t)p.tab.total * sizeof(float2); }
  __device__ static const float4* global_table(const Params& p) {
    if constexpr (kInline) return p.v;
    else return reinterpret_cast<const float4*>(p.tab.coef);
  }

  __device__ static void stage(const Params& p, float4* s) {
    if constexpr (!kInline) {
      const float4* src = reinterpret_cast<const float4*>(p.tab.coef);
      for (uint32_t i = threadIdx.x; i < p.tab.total / 2; i += blockDim.x) s[i] = src[i];
    }
  }

  // Two groups that bound the coordinate w as a function of the other one, v
  // (lo: max-reduced, hi: min-reduced), consumed in lockstep so each iteration
  // carries 4 edges x P points of work. The seeds wlo / whi enter as the free
  // third operand of the first FMNMX3 (prep.cu guarantees >= 1 pair per
  // group). With wlo = whi = w, afterwards lo >= w >= hi and the point
  // satisfies the section iff lo <= hi.
  __device__ __forceinline__ static void section(const float4* A, uint32_t na, const float4* B,
                                                 uint32_t nb, const float (&v)[P],
                                                 const float (&wlo)[P], const float (&whi)[P],
                                                 float (&lo)[P], float (&hi)[P]) {
    {
      const float4 a = A[0], b = B[0];
#pragma unroll
      for (int p = 0; p < P; ++p) {
        lo[p] = fmax3(wlo[p], fmaf(a.x, v[p], a.y), fmaf(a.z, v[p], a.w));
        hi[p] = fmin3(whi[p], fmaf(b.x, v[p], b.y), fmaf(b.z, v[p], b.w));
      }
    }
    const uint32_t nc = na < nb ? na : nb;
    uint32_t i = 1;
    VPIPG_UNROLL(VPIPG_SLAB_UNROLL)
    for (; i < nc; ++i) {
      const float4 a = A[i], b = B[i];
#pragma unroll
      for (int p = 0; p < P; ++p) {
        lo[p] = fmax3(lo[p], fmaf(a.x, v[p], a.y), fmaf(a.z, v[p], a.w));
        hi[p] = fmin3(hi[p], fmaf(b.x, v[p], b.y), fmaf(b.z, v[p], b.w));
      }
    }
#pragma unroll 1
    for (uint32_t j = i; j < na; ++j) {
      const float4 a = A[j];
#pragma unroll
      for (int p = 0; p < P; ++p) lo[p] = fmax3(lo[p], fmaf(a.x, v[p], a.y), fmaf(a.z, v[p], a.w));
    }
#pragma unroll 1
    for (uint32_t j = i; j < nb; ++j) {
      const float4 b = B[j];
#pragma unroll
      for (int p = 0; p < P; ++p) hi[p] = fmin3(hi[p], fmaf(b.x, v[p], b.y), fmaf(b.z, v[p], b.w));
    }
  }

  // Point p is inside iff a[p] >= b[p] (every half-plane holds; ties inside).
  // Most tables have one section (prep.cu: every edge expressed as a bound on
  // y, or every edge on x): lo >= w >= hi, inside iff lo <= hi. Otherwise
  // section 1 (x bounded by lines in y) leaves lo1 >= x >= hi1 with the
  // violation f1 = lo1 - hi1 >= 0, zero iff the point satisfies it. Section 2
  // is seeded with lo = y + f1, hi = y, so its lo <= hi test also fails when
  // section 1 did: y + f1 > y for every f1 that survives rounding against y,
  // and an f1 below half an ulp of y is a violation of < 6e-8 |y|, inside the
  // 1e-5 band. One compare per point decides both sections.
  __device__ __forceinline__ static void eval(const Params& prm, const float4* s,
                                              const float (&x)[P], const float (&y)[P],
                                              float (&a)[P], float (&b)[P]) {
    const SlabTable& t = prm.tab;
    float lo[P], hi[P];
    // single-section tables: y alone, bounded by lines in x (mode 1), or x
    // alone, bounded by lines in y (mode 2)
    auto y_only = [&] {
      section(s + t.off[2] / 2, t.cnt[2] / 2, s + t.off[3] / 2, t.cnt[3] / 2, x, y, y, lo, hi);
    };
    auto x_only = [&] {
      section(s + t.off[0] / 2, t.cnt[0] / 2, s + t.off[1] / 2, t.cnt[1] / 2, y, x, x, lo, hi);
    };
    auto mixed = [&] {
      section(s + t.off[0] / 2, t.cnt[0] / 2, s + t.off[1] / 2, t.cnt[1] / 2, y, x, x, lo, hi);
      float seed[P];
#pragma unroll
      for (int p = 0; p < P; ++p) seed[p] = y[p] + (lo[p] - hi[p]);
      section(s + t.off[2] / 2, t.cnt[2] / 2, s + t.off[3] / 2, t.cnt[3] / 2, x, seed, y, lo, hi);
    };
    if constexpr (kMode == 0) {
      mixed();
    } else if constexpr (kMode == 1) {
      y_only();
    } else if constexpr (kMode == 2) {
      x_only();
    } else {
      if (t.cnt[0] == 0) y_only();
      else if (t.cnt[2] == 0) x_only();
      else mixed();
    }
#pragma unroll
    for (int p = 0; p < P; ++p) {
      a[p] = hi[p];
      b[p] = lo[p];
    }
  }
};

struct CrossParams {
  CrossTable tab;
  float ox, oy;
};
struct CrossParamsInl {
  CrossTable tab;
  float ox, oy;
  float4 v[kInlineMax];
};

template <int P, bool kInline = false>
struct CrossEngine {
  static constexpr int kP = P;
  static constexpr bool kInl = kInline;
  // the uniform round loop (ldg_kernel): with parameter-bank tables the edge
  // loop runs on uniform registers; with shared-memory tables (n > kInlineMax)
  // it measured faster too (c3x:256 crossing 10.36 vs 11.27 ms)
  static constexpr bool kUniform = true;
  // parameter-bank tables are handed over in the absolute frame (the host
  // adds the origin back, launch_test_f32): the crossing's f32 arithmetic is
  // accurate to an ulp of the coordinates there (h and g are exact near the
  // polygon, Sterbenz), and a per-point shift right after the loads measured
  // 7 % slower on C5 (11.09 vs 10.35 ms); shared-memory tables stay local
  static constexpr bool kShiftIn = VPIPG_LOCAL_FRAME && !kInline;
  static constexpr int kVote = VPIPG_CROSS_VOTE;  // 2: a holds the parity word, sign bit = inside
#ifndef VPIPG_CROSS_LDG
#define VPIPG_CROSS_LDG 1
#endif
  // 1: ldg_kernel (register streaming), 0: stream_kernel (per-warp TMA ring);
  // with parameter-bank tables the ring's barrier loops keep the compiler from
  // using the uniform datapath in the edge loop (C5: 12.32 vs 11.20 ms)
  static constexpr bool kRegStream = VPIPG_CROSS_LDG;
  using Params = std::conditional_t<kInline, CrossParamsInl, CrossParams>;
  static size_t table_bytes(const Params& p) { return kInline ? 0 : (size_t)p.tab.n * sizeof(float4); }
  __device__ static const float4* global_table(const Params& p) {
    if constexpr (kInline) return p.v;
    else return p.tab.vert;
  }

  __device__ static void stage(const Params& p, float4* s) {
    if constexpr (!kInline)
      for (uint32_t i = threadIdx.x; i < p.tab.n; i += blockDim.x) s[i] = p.tab.vert[i];
  }

  // a[p]: the parity word (sign bit set = odd crossing count = inside), b[p] = 0
  __device__ __forceinline__ static void eval(const Params& prm, const float4* s,
                                              const float (&x)[P], const float (&y)[P],
                                              float (&a)[P], float (&b)[P]) {
    const uint32_t n = prm.tab.n;
    uint32_t par[P];
#pragma unroll
    for (int p = 0; p < P; ++p) par[p] = 0;
    // record k = (u.x, u.y, dvx/dvy, -) of edge w = v[k-1] -> u = v[k] (prep.cu)
    if (n > 0) {
      const float4 last = s[n - 1];
      float hp[P];  // h of the vertex before the current pair
#pragma unroll
      for (int p = 0; p < P; ++p) hp[p] = y[p] - last.y;
      uint32_t k = 0;
      VPIPG_UNROLL(VPIPG_CROSS_UNROLL)
      for (; k + 3 < n; k += 4) {
        const float4 v0 = s[k], v1 = s[k + 1], v2 = s[k + 2], v3 = s[k + 3];
#pragma unroll
        for (int p = 0; p < P; ++p) {
          const float h0 = y[p] - v0.y, g0 = v0.x - x[p];
          const float h1 = y[p] - v1.y;
          const float h2 = y[p] - v2.y, g2 = v2.x - x[p];
          const float h3 = y[p] - v3.y;
          const uint32_t t0 = cross_bit(h0, hp[p], fmaf(h0, v0.z, g0));  // u-anchored at v[k]
          const uint32_t t1 = cross_bit(h1, h0, fmaf(h0, v1.z, g0));     // w-anchored at v[k]
          const uint32_t t2 = cross_bit(h2, h1, fmaf(h2, v2.z, g2));
          const uint32_t t3 = cross_bit(h3, h2, fmaf(h2, v3.z, g2));
          par[p] ^= t0 ^ t1 ^ t2 ^ t3;
          hp[p] = h3;
        }
      }
      if (k + 1 < n) {
        const float4 v0 = s[k], v1 = s[k + 1];
#pragma unroll
        for (int p = 0; p < P; ++p) {
          const float h0 = y[p] - v0.y, g0 = v0.x - x[p];
          const float h1 = y[p] - v1.y;
          par[p] ^= cross_bit(h0, hp[p], fmaf(h0, v0.z, g0)) ^ cross_bit(h1, h0, fmaf(h0, v1.z, g0));
          hp[p] = h1;
        }
        k += 2;
      }
      if (k < n) {
        const float4 v0 = s[k];
#pragma unroll
        for (int p = 0; p < P; ++p) {
          const float h0 = y[p] - v0.y;
          par[p] ^= cross_bit(h0, hp[p], fmaf(h0, v0.z, v0.x - x[p]));
        }
      }
    }
#pragma unroll
    for (int p = 0; p < P; ++p) {
      if (kVote == 2) {
        a[p] = __uint_as_float(par[p]);
      } else {
        a[p] = __uint_as_float((~par[p] & 0x80000000u) | 0x3f800000u);
      }
      b[p] = 0.f;
    }
  }
};

// live == false (a warp whose slot in the last round is past the end; warp-
// uniform): the votes run, nothing is stored or counted
template <bool kGuard, int kVote, int P>
__device__ __forceinline__ cnt_t emit(float (&av)[P], const float (&bv)[P], uint64_t base,
                                         const TestArgs& a, int lane, bool live = true) {
  static_assert(kGuard || P % 4 == 0, "16-byte word stores need P % 4 == 0");
  uint32_t w[P];
  cnt_t cnt = 0;
#pragma unroll
  for (int p = 0; p < P; ++p) {
    if (kGuard && base + 32u * p + lane >= a.m) av[p] = kVote == 2 ? 0.f : -INFINITY;
    w[p] = vote_in<kVote>(av[p], bv[p], cnt);
  }
  if (!live) return 0;
  if (a.words && lane == 0) {
    const uint64_t w0 = base >> 5;
    if (!kGuard && (reinterpret_cast<uintptr_t>(a.words) & 15) == 0) {
      uint4* dst = reinterpret_cast<uint4*>(a.words + w0);
#pragma unroll
      for (int q = 0; q < P / 4; ++q) __stcs(dst + q, make_uint4(w[4 * q], w[4 * q + 1], w[4 * q + 2], w[4 * q + 3]));
    } else {
      const uint64_t nwords = (a.m + 31) >> 5;
#pragma unroll
      for (int p = 0; p < P; ++p)
        if (!kGuard || w0 + p < nwords) a.words[w0 + p] = w[p];
    }
  }
  if (a.bytes) {
#pragma unroll
    for (int p = 0; p < P; ++p) {
      const uint64_t idx = base + 32u * p + lane;
      if (!kGuard || idx < a.m) a.bytes[idx] = (w[p] >> lane) & 1u;
    }
  }
  return cnt;
}

// Guarded warp tile straight from global memory (tails, unaligned inputs).
template <class Eng, bool kShift = Eng::kShiftIn>
__device__ __forceinline__ cnt_t guarded_tile(const typename Eng::Params& prm, const float4* tab,
                                                 const TestArgs& a, uint64_t base, int lane) {
  constexpr int P = Eng::kP;
  const float* xs = static_cast<const float*>(a.xs);
  const float* ys = static_cast<const float*>(a.ys);
  float x[P], y[P], va[P], vb[P];
#pragma unroll
  for (int p = 0; p < P; ++p) {
    const uint64_t idx = base + 32u * p + lane;
    const bool ok = idx < a.m;
    x[p] = ok ? __ldcs(xs + idx) : 0.f;
    y[p] = ok ? __ldcs(ys + idx) : 0.f;
  }
  if constexpr (kShift) to_local(x, y, prm.ox, prm.oy);
  Eng::eval(prm, tab, x, y, va, vb);
  return emit<true, Eng::kVote, P>(va, vb, base, a, lane);
}

// kSmemTab: the polygon table is staged in shared memory once per CTA (the
// normal case); polygons whose table exceeds kSmemTableMax read it from global
// memory with warp-uniform loads instead.
template <class Eng, bool kSmemTab>
__global__ void __launch_bounds__(kThreads, 2)
    stream_kernel(const __grid_constant__ typename Eng::Params prm, const TestArgs a,
                  const uint64_t full_slices) {
  constexpr int P = Eng::kP;
  constexpr int kWarpPts = 32 * P;
  extern __shared__ __align__(128) unsigned char smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // per-warp ring: [stage][x | y][kWarpPts] floats, then the barriers, then the table
  float* ring = reinterpret_cast<float*>(smem) + (size_t)warp * kStages * 2 * kWarpPts;
  uint64_t* bars = reinterpret_cast<uint64_t*>(reinterpret_cast<float*>(smem) +
                                               (size_t)kWarps * kStages * 2 * kWarpPts);
  uint64_t* full = bars + warp * 2 * kStages;
  uint64_t* empty = full + kStages;
  float4* s_tab = reinterpret_cast<float4*>(bars + kWarps * 2 * kStages);
  if (lane == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 32);
    }
    mbar_fence_init();
  }
  if (kSmemTab) Eng::stage(prm, s_tab);
  const float4* tab = (kSmemTab && !Eng::kInl) ? s_tab : Eng::global_table(prm);
  __syncthreads();

  const SliceRounds sr(full_slices, warp);
  const float* xs = static_cast<const float*>(a.xs);
  const float* ys = static_cast<const float*>(a.ys);
  uint64_t policy = 0;
  if (lane == 0) {
    policy = policy_evict_first();
    for (int s = 0; s < kStages; ++s) {
      if (s >= sr.rounds) break;
      const uint64_t g = sr.slice(s);
      mbar_arrive_expect_tx(&full[s], 2u * kWarpPts * sizeof(float));
      bulk_g2s(ring + s * 2 * kWarpPts, xs + g * kWarpPts, kWarpPts * sizeof(float), &full[s], policy);
      bulk_g2s(ring + s * 2 * kWarpPts + kWarpPts, ys + g * kWarpPts, kWarpPts * sizeof(float),
               &full[s], policy);
    }
  }
  cnt_t count = 0;
  for (uint64_t r = 0; r < sr.rounds; ++r) {
    const uint32_t s = r % kStages, ph = (r / kStages) & 1u;
    mbar_wait(&full[s], ph);
    const float* px = ring + s * 2 * kWarpPts + lane;
    float x[P], y[P], va[P], vb[P];
#pragma unroll
    for (int p = 0; p < P; ++p) {
      x[p] = px[32 * p];
      y[p] = px[kWarpPts + 32 * p];
    }
    if constexpr (Eng::kShiftIn) to_local(x, y, prm.ox, prm.oy);
    mbar_arrive(&empty[s]);  // release: this lane's reads of stage s are done
    if (lane == 0 && r + kStages < sr.rounds) {
      const uint64_t gn = sr.slice(r + kStages);
      mbar_wait(&empty[s], ph);
      mbar_arrive_expect_tx(&full[s], 2u * kWarpPts * sizeof(float));
      bulk_g2s(ring + s * 2 * kWarpPts, xs + gn * kWarpPts, kWarpPts * sizeof(float), &full[s], policy);
      bulk_g2s(ring + s * 2 * kWarpPts + kWarpPts, ys + gn * kWarpPts, kWarpPts * sizeof(float),
               &full[s], policy);
    }
    Eng::eval(prm, tab, x, y, va, vb);
    count += emit<false, Eng::kVote, P>(va, vb, sr.slice(r) * kWarpPts, a, lane, sr.live(r));
  }
  // partial last slice: the warp next in round-robin order, guarded loads
  if (sr.g0 == full_slices % sr.W) {
    for (uint64_t base = full_slices * kWarpPts; base < a.m; base += kWarpPts)
      count += guarded_tile<Eng>(prm, tab, a, base, lane);
  }
  flush_count(count, a);
}

// Register-streaming variant (the slab engines): no shared-memory ring -- each
// warp loads its slice straight into registers (coalesced 128-byte rows,
// evict-first) after an L2 prefetch of the slice two rounds ahead. Measured
// against the TMA ring: equal at C5 (compute-bound), 7 % faster at C3 n = 8
// (memory-bound: 6.6 TB/s), so the slab engines use it; the crossing engine
// keeps the ring (3 % faster there).
#ifndef VPIPG_LDG_MINB
#define VPIPG_LDG_MINB 2
#endif
template <class Eng, bool kSmemTab>
__global__ void __launch_bounds__(kThreads, VPIPG_LDG_MINB)
    ldg_kernel(const __grid_constant__ typename Eng::Params prm, const TestArgs a,
               const uint64_t full_slices) {
  constexpr int P = Eng::kP;
  constexpr int kWarpPts = 32 * P;
  extern __shared__ __align__(128) unsigned char smem[];
  float4* s_tab = reinterpret_cast<float4*>(smem);
  if (kSmemTab) Eng::stage(prm, s_tab);
  const float4* tab = (kSmemTab && !Eng::kInl) ? s_tab : Eng::global_table(prm);
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const SliceRounds sr(full_slices, warp);
  const float* xs = static_cast<const float*>(a.xs);
  const float* ys = static_cast<const float*>(a.ys);
  constexpr int kLines = kWarpPts * 4 / 128;
  auto prefetch = [&](uint64_t r) {
    if (r >= sr.rounds) return;
    const uint64_t g = sr.slice(r);
    for (int l = lane; l < 2 * kLines; l += 32)
      prefetch_l2((l < kLines ? xs : ys) + g * kWarpPts + (l % kLines) * 32);
  };
#ifndef VPIPG_PF_AHEAD
#define VPIPG_PF_AHEAD 1
#endif
  cnt_t count = 0;
  // the uniform round loop only pays where the edge loop reads the parameter
  // bank through uniform registers (the crossing engine); the slab engines'
  // FFMAs take two table operands, so they read the table into vector
  // registers either way and keep the plain strided loop (C5: 5.24 vs 5.35 ms)
#ifndef VPIPG_SLICE_ROUNDS
#define VPIPG_SLICE_ROUNDS 0
#endif
  if constexpr (Eng::kUniform || VPIPG_SLICE_ROUNDS) {
    for (int d = 0; d < VPIPG_PF_AHEAD; ++d) prefetch(d);
    for (uint64_t r = 0; r < sr.rounds; ++r) {
      prefetch(r + VPIPG_PF_AHEAD);
      const uint64_t g = sr.slice(r);
      const float* px = xs + g * kWarpPts + lane;
      const float* py = ys + g * kWarpPts + lane;
      float x[P], y[P], va[P], vb[P];
#pragma unroll
      for (int p = 0; p < P; ++p) {
        x[p] = __ldcs(px + 32 * p);
        y[p] = __ldcs(py + 32 * p);
      }
      if constexpr (Eng::kShiftIn) to_local(x, y, prm.ox, prm.oy);
      Eng::eval(prm, tab, x, y, va, vb);
      count += emit<false, Eng::kVote, P>(va, vb, g * kWarpPts, a, lane, sr.live(r));
    }
  } else {
    auto pf = [&](uint64_t g) {
      if (g >= full_slices) return;
      for (int l = lane; l < 2 * kLines; l += 32)
        prefetch_l2((l < kLines ? xs : ys) + g * kWarpPts + (l % kLines) * 32);
    };
    pf(sr.g0);
    for (uint64_t g = sr.g0; g < full_slices; g += sr.W) {
      pf(g + sr.W);
      const float* px = xs + g * kWarpPts + lane;
      const float* py = ys + g * kWarpPts + lane;
      float x[P], y[P], va[P], vb[P];
#pragma unroll
      for (int p = 0; p < P; ++p) {
        x[p] = __ldcs(px + 32 * p);
        y[p] = __ldcs(py + 32 * p);
      }
      if constexpr (Eng::kShiftIn) to_local(x, y, prm.ox, prm.oy);
      Eng::eval(prm, tab, x, y, va, vb);
      count += emit<false, Eng::kVote, P>(va, vb, g * kWarpPts, a, lane);
    }
  }
  if (sr.g0 == full_slices % sr.W) {
    for (uint64_t base = full_slices * kWarpPts; base < a.m; base += kWarpPts)
      count += guarded_tile<Eng>(prm, tab, a, base, lane);
  }
  flush_count(count, a);
}

// ---------------------------------------------------------------------------
// Fused three-engine pass (vpipg_test_multi with all engines, fp32): every
// point is read once and tested by Voronoi, sign-of-offset and crossing in
// turn, each writing its own mask words and count. Same slice schedule and
// loads as ldg_kernel; the three tables sit side by side in shared memory.
// the three engines' live registers set P: 16 (C5 fused 19.47 ms; 12: 20.52,
// 20: 19.87 with spills)
#ifndef VPIPG_TRI_P
#define VPIPG_TRI_P 16
#endif
constexpr int kTriP = VPIPG_TRI_P;
struct TriParams {
  SlabParams v, o;
  CrossParams c;
  uint32_t off_o, off_c;  // float4 offsets of the offset / crossing tables in shared memory
};
constexpr int kTriInlineMax = 256;
struct TriParamsInl {   // the three tables in the parameter bank (VPIPG_INLINE)
  SlabParams v, o;
  CrossParams c;
  uint32_t off_o, off_c;  // float4 offsets of the offset / crossing tables in `t`
  float4 t[kTriInlineMax];
};

// kMode: the slab table form shared by the Voronoi and offset tables (their
// lines coincide: each bisector is the edge line), -1 when they differ
// VPIPG_TRI_SLAB_SMEM: with parameter-bank tables, the two slab tables still
// staged in shared memory (LDS.128 into vector registers, as the per-engine
// slab kernels) and only the crossing table read as uniform registers
#ifndef VPIPG_TRI_SLAB_SMEM
#define VPIPG_TRI_SLAB_SMEM 1
#endif
#ifndef VPIPG_TRI_MINB
#define VPIPG_TRI_MINB 2
#endif
template <int kMode, bool kInline = false>
__global__ void __launch_bounds__(kThreads, VPIPG_TRI_MINB)
    tri_kernel(const __grid_constant__ std::conditional_t<kInline, TriParamsInl, TriParams> prm,
               const TestArgs av, const TestArgs ao, const TestArgs ac, const uint64_t full_slices) {
  using TriV = SlabEngine<kTriP, false, kMode>;
  using TriO = SlabEngine<kTriP, true, kMode>;
  using TriC = CrossEngine<kTriP>;
  // one set of register-streamed loads feeds all three engines
  static_assert(TriV::kRegStream && TriO::kRegStream, "slab engines stream through registers");
  constexpr int P = kTriP;
  constexpr int kWarpPts = 32 * P;
  extern __shared__ __align__(128) unsigned char smem[];
  float4* s_tab = reinterpret_cast<float4*>(smem);
  const float4* tv;
  const float4* tc;
  if constexpr (kInline && !VPIPG_TRI_SLAB_SMEM) {
    (void)s_tab;
    tv = prm.t;
    tc = prm.t + prm.off_c;
  } else {
    TriV::stage(prm.v, s_tab);
    TriO::stage(prm.o, s_tab + prm.off_o);
    tv = s_tab;
    if constexpr (kInline) {
      tc = prm.t + prm.off_c;
    } else {
      TriC::stage(prm.c, s_tab + prm.off_c);
      tc = s_tab + prm.off_c;
    }
  }
  const float4* to = tv + prm.off_o;
  __syncthreads();
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
  prefetch(0);
  for (uint64_t r = 0; r < sr.rounds; ++r) {
    prefetch(r + 1);
    const uint64_t g = sr.slice(r);
    const bool live = sr.live(r);
    const float* px = xs + g * kWarpPts + lane;
    const float* py = ys + g * kWarpPts + lane;
    float x[P], y[P], va[P], vb[P];
#pragma unroll
    for (int p = 0; p < P; ++p) {
      x[p] = __ldcs(px + 32 * p);
      y[p] = __ldcs(py + 32 * p);
    }
    // the crossing engine first, on the points as loaded with its parameter-
    // bank table in the absolute frame (exactly the standalone kernel's
    // arithmetic, so both routes give the same masks); then the points move to
    // the local frame for the slab engines
    if constexpr (kInline) {
      TriC::eval(prm.c, tc, x, y, va, vb);
      cc += emit<false, TriC::kVote, P>(va, vb, g * kWarpPts, ac, lane, live);
    }
    to_local(x, y, prm.v.ox, prm.v.oy);
    TriV::eval(prm.v, tv, x, y, va, vb);
    cv += emit<false, TriV::kVote, P>(va, vb, g * kWarpPts, av, lane, live);
    TriO::eval(prm.o, to, x, y, va, vb);
    co += emit<false, TriO::kVote, P>(va, vb, g * kWarpPts, ao, lane, live);
    if constexpr (!kInline) {
      TriC::eval(prm.c, tc, x, y, va, vb);
      cc += emit<false, TriC::kVote, P>(va, vb, g * kWarpPts, ac, lane, live);
    }
  }
  if (sr.g0 == full_slices % sr.W) {
    for (uint64_t base = full_slices * kWarpPts; base < av.m; base += kWarpPts) {
      cv += guarded_tile<TriV>(prm.v, tv, av, base, lane);
      co += guarded_tile<TriO>(prm.o, to, ao, base, lane);
      cc += guarded_tile<TriC, !kInline>(prm.c, tc, ac, base, lane);
    }
  }
  flush_count(cv, av);
  flush_count(co, ao);
  flush_count(cc, ac);
}

template <class Eng, bool kSmemTab>
__global__ void __launch_bounds__(kThreads) generic_kernel(const __grid_constant__ typename Eng::Params prm,
                                                          const TestArgs a) {
  constexpr int kWarpPts = 32 * Eng::kP;
  extern __shared__ __align__(16) float4 s_gtab[];
  if (kSmemTab) {
    Eng::stage(prm, s_gtab);
    __syncthreads();
  }
  const float4* gtab = (kSmemTab && !Eng::kInl) ? s_gtab : Eng::global_table(prm);
  const int lane = threadIdx.x & 31;
  const uint64_t gwarp = (uint64_t)blockIdx.x * (kThreads / 32) + (threadIdx.x >> 5);
  cnt_t count = 0;
  for (uint64_t base = gwarp * kWarpPts; base < a.m;
       base += (uint64_t)gridDim.x * (kThreads / 32) * kWarpPts)
    count += guarded_tile<Eng>(prm, gtab, a, base, lane);
  flush_count(count, a);
}


constexpr size_t kSmemTableMax = 96 * 1024;


template <class Eng>
cudaError_t launch(const typename Eng::Params& prm, const TestArgs& a, cudaStream_t stream) {
  constexpr int kWarpPts = 32 * Eng::kP;
  const bool staged = Eng::table_bytes(prm) <= kSmemTableMax;
  const size_t tab = staged ? Eng::table_bytes(prm) : 0;
  const bool aligned = ((reinterpret_cast<uintptr_t>(a.xs) | reinterpret_cast<uintptr_t>(a.ys)) & 15) == 0;
  const uint64_t full_slices = aligned ? a.m / kWarpPts : 0;
  if (full_slices < kWarps) {
    auto k = staged ? generic_kernel<Eng, true> : generic_kernel<Eng, false>;
    int sms = 0, per_sm = 0;
    cudaError_t e = launch_config(reinterpret_cast<const void*>(k), kThreads, tab, &sms, &per_sm);
    if (e != cudaSuccess) return e;
    const uint64_t warps = (a.m + kWarpPts - 1) / kWarpPts;
    const uint64_t blocks = (warps + kThreads / 32 - 1) / (kThreads / 32);
    const uint64_t cap = (uint64_t)sms * 4;
    k<<<(int)(blocks < cap ? blocks : cap), kThreads, tab, stream>>>(prm, a);
    return cudaGetLastError();
  }
  using Kernel = void (*)(const typename Eng::Params, const TestArgs, const uint64_t);
  Kernel k;
  size_t smem;
  if constexpr (Eng::kRegStream) {
    k = staged ? ldg_kernel<Eng, true> : ldg_kernel<Eng, false>;
    smem = tab;
  } else {
    k = staged ? stream_kernel<Eng, true> : stream_kernel<Eng, false>;
    smem = (size_t)kWarps * kStages * 2 * kWarpPts * sizeof(float) +
           (size_t)kWarps * 2 * kStages * sizeof(uint64_t) + tab;
  }
  int sms = 0, per_sm = 0;
  cudaError_t e = launch_config(reinterpret_cast<const void*>(k), kThreads, smem, &sms, &per_sm);
  if (e != cudaSuccess) return e;
  const uint64_t cap = (uint64_t)sms * per_sm;
  const uint64_t want = (full_slices + kWarps - 1) / kWarps;
  const int grid = (int)(want < cap ? want : cap);
  k<<<grid, kThreads, smem, stream>>>(prm, a, full_slices);
  return cudaGetLastError();
}

}  // namespace

// Polygons with more edges than this run the per-engine kernels even when all
// three engines are asked for. With parameter-bank tables the fused kernel
// stays 4-6 % ahead of the three per-engine kernels up to n = 96 on the
// exact-n c3x polygons (2^28 points: n = 40 2.95 vs 3.12 ms, 64 4.52 vs 4.8,
// 96 6.63; profiles/sweep_r02.json); past that its tables no longer fit the
// parameter bank (kTriInlineMax float4 records)
#ifndef VPIPG_FUSE_MAX_N
#define VPIPG_FUSE_MAX_N 96
#endif

float4 cross_record_abs(const float4& r, float ox, float oy) {
  return make_float4(static_cast<float>(static_cast<double>(r.x) + ox),
                     static_cast<float>(static_cast<double>(r.y) + oy), r.z,
                     static_cast<float>(static_cast<double>(r.w) + ox));
}

bool test_f32_all_plan(const DevTables& t, const TestArgs* a, size_t* smem_out) {
  if (test_f32_small_plan(t, a)) {
    if (smem_out) *smem_out = 0;
    return true;
  }
  constexpr int kWarpPts = 32 * kTriP;
  const size_t smem = ((size_t)t.slab[0].total / 2 + (size_t)t.slab[1].total / 2 + t.cross.n) *
                      sizeof(float4);
  const bool aligned =
      ((reinterpret_cast<uintptr_t>(a[0].xs) | reinterpret_cast<uintptr_t>(a[0].ys)) & 15) == 0;
  const uint64_t full_slices = aligned ? a[0].m / kWarpPts : 0;
  if (smem_out) *smem_out = smem;
  return t.cross.n <= VPIPG_FUSE_MAX_N && smem <= kSmemTableMax && full_slices >= kWarps;
}

cudaError_t launch_test_f32_all(const DevTables& t, const TestArgs* a, cudaStream_t stream) {
  using TriV = SlabEngine<kTriP, false>;
  using TriO = SlabEngine<kTriP, true>;
  constexpr int kWarpPts = 32 * kTriP;
  const cudaError_t es = launch_test_f32_small(t, a, stream);
  if (es != cudaErrorNotSupported) return es;
  if (!test_f32_all_plan(t, a, nullptr)) return cudaErrorNotSupported;
  TriParams prm{};
  prm.v = TriV::Params{t.slab[0], t.ox, t.oy};
  prm.o = TriO::Params{t.slab[1], t.ox, t.oy};
  prm.c = CrossParams{t.cross, t.ox, t.oy};
  const size_t nv = TriV::table_bytes(prm.v) / sizeof(float4);
  const size_t no = TriO::table_bytes(prm.o) / sizeof(float4);
  const size_t nc = CrossEngine<kTriP>::table_bytes(prm.c) / sizeof(float4);
  prm.off_o = static_cast<uint32_t>(nv);
  prm.off_c = static_cast<uint32_t>(nv + no);
  const bool inl = VPIPG_INLINE && t.h_cross && t.h_slab[0] && t.h_slab[1] && nv + no + nc <= kTriInlineMax;
  const size_t smem = inl ? (VPIPG_TRI_SLAB_SMEM ? (nv + no) * sizeof(float4) : 0)
                          : (nv + no + nc) * sizeof(float4);
  const uint64_t full_slices = a[0].m / kWarpPts;
  int sms = 0, per_sm = 0;
  auto form = [](const SlabTable& t) { return t.cnt[0] == 0 ? 1 : t.cnt[2] == 0 ? 2 : 0; };
  const int fv = form(t.slab[0]), fo = form(t.slab[1]);
  const int mode = fv == fo ? fv : -1;
  auto go = [&](auto il, const auto& params) -> cudaError_t {
    constexpr bool I = decltype(il)::value;
    auto kern = mode == 0 ? tri_kernel<0, I> : mode == 1 ? tri_kernel<1, I>
              : mode == 2 ? tri_kernel<2, I> : tri_kernel<-1, I>;
    cudaError_t e = launch_config(reinterpret_cast<const void*>(kern), kThreads, smem, &sms, &per_sm);
    if (e != cudaSuccess) return e;
    const uint64_t cap = (uint64_t)sms * per_sm;
    const uint64_t want = (full_slices + kWarps - 1) / kWarps;
    const int grid = (int)(want < cap ? want : cap);
    kern<<<grid, kThreads, smem, stream>>>(params, a[0], a[1], a[2], full_slices);
    return cudaGetLastError();
  };
  if (inl) {
    TriParamsInl pi{};
    pi.v = prm.v;
    pi.o = prm.o;
    pi.c = prm.c;
    pi.off_o = prm.off_o;
    pi.off_c = prm.off_c;
    std::memcpy(pi.t, t.h_slab[0], nv * sizeof(float4));
    std::memcpy(pi.t + nv, t.h_slab[1], no * sizeof(float4));
    for (size_t k = 0; k < nc; ++k) pi.t[nv + no + k] = cross_record_abs(t.h_cross[k], t.ox, t.oy);
    return go(std::true_type{}, pi);
  }
  return go(std::false_type{}, prm);
}

template <bool kNanIn, int kMode>
cudaError_t launch_slab_mode(const DevTables& t, int engine, const TestArgs& a, cudaStream_t stream) {
#ifndef VPIPG_SLAB_INLINE
#define VPIPG_SLAB_INLINE 0
#endif
  if (VPIPG_SLAB_INLINE && t.h_slab[engine] && t.slab[engine].total / 2 <= (uint32_t)kInlineMax) {
    using E = SlabEngine<VPIPG_SLAB_P, kNanIn, kMode, true>;
    typename E::Params prm{};
    prm.tab = t.slab[engine];
    prm.ox = t.ox;
    prm.oy = t.oy;
    std::memcpy(prm.v, t.h_slab[engine], t.slab[engine].total * sizeof(float2));
    return launch<E>(prm, a, stream);
  }
  using E = SlabEngine<VPIPG_SLAB_P, kNanIn, kMode>;
  typename E::Params prm{t.slab[engine], t.ox, t.oy};
  return launch<E>(prm, a, stream);
}

template <bool kNanIn>
cudaError_t launch_slab(const DevTables& t, int engine, const TestArgs& a, cudaStream_t stream) {
  const SlabTable& tab = t.slab[engine];
  if (tab.cnt[0] == 0) return launch_slab_mode<kNanIn, 1>(t, engine, a, stream);
  if (tab.cnt[2] == 0) return launch_slab_mode<kNanIn, 2>(t, engine, a, stream);
  return launch_slab_mode<kNanIn, 0>(t, engine, a, stream);
}

cudaError_t launch_test_f32(const DevTables& t, int engine, const TestArgs& a,
                            cudaStream_t stream) {
  if (engine == 0) return launch_slab<false>(t, 0, a, stream);
  if (engine == 1) return launch_slab<true>(t, 1, a, stream);
  if (VPIPG_INLINE && t.h_cross && t.cross.n <= (uint32_t)kInlineMax) {
    CrossParamsInl prm{};
    prm.tab = t.cross;
    prm.ox = t.ox;
    prm.oy = t.oy;
    for (uint32_t k = 0; k < t.cross.n; ++k) prm.v[k] = cross_record_abs(t.h_cross[k], t.ox, t.oy);
    return launch<CrossEngine<VPIPG_CROSS_P, true>>(prm, a, stream);
  }
  return launch<CrossEngine<VPIPG_CROSS_P>>(CrossParams{t.cross, t.ox, t.oy}, a, stream);
}

}  // namespace vpipg
