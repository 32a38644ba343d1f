// prep.cu -- polygon preprocessing kernel (the device half of vpipg_prepare).
//
// Replaces the reference's conversion step: centroid (geometry.cpp:106-120),
// edge_coefficients (voronoi.cpp:23-31) and reflect_generator
// (voronoi.cpp:46-58) composed by to_voronoi (voronoi.cpp:60-71), plus the
// per-edge setup the reference batch kernels hoist out of their point loops
// (engines.cpp:146-149, :176-186). One CTA per polygon.
//
// The f64 outputs (generators, offset and ray records) repeat the
// reference's expressions operation for operation with explicitly rounded
// intrinsics (__dmul_rn / __dadd_rn / __dsub_rn / __ddiv_rn are never
// contracted into FMAs), so they are bit-identical to the reference's
// -ffp-contract=off build. The fp32 slab tables are derived from those f64
// values (accuracy matters there, bit-matching does not).
#include <climits>
#include <cmath>
#include <cstdint>

#include "exact_geom.cuh"
#include "vpipg_device.cuh"
#include "vpipg_internal.h"

namespace vpipg {

namespace {

constexpr int kPrepThreads = 256;
enum : int { kNone = -1, kXlo = 0, kXhi = 1, kYlo = 2, kYhi = 3 };


// Half-plane a*x' + b*y' + c >= 0 (local frame) -> slab class and (B, C),
// under one of three orientation modes:
//   kMixed   |a| >= |b| -> x-bound (x' >= / <= B y' + C), else y-bound, so
//            |B| <= 1 (the general case: two sections, chained seed);
//   kPreferY every edge is a y-bound unless it is within 2^-VPIPG_SLAB_STEEP
//            rad of vertical;
//   kPreferX the transpose.
// A polygon with no such near-vertical (near-horizontal) edge has empty x (y)
// groups under kPreferY (kPreferX) and the test kernels run ONE section with
// no chained seed; slab_scatter picks the cheaper of the two when either
// applies. Precision: the f32 FFMA and the rounding of B and C misplace the
// line by about 1.2e-7 (|v'| + |C / B|) in distance whatever |B| is (C / B is
// the line's intercept, within the polygon's extent of the frame origin for
// the lines that matter), far inside the 1e-5 band; the cap on |B| keeps
// B v' finite for any f32 point of interest.
#ifndef VPIPG_SLAB_STEEP
#define VPIPG_SLAB_STEEP 16
#endif
enum : int { kMixed = 0, kPreferY = 1, kPreferX = 2 };
__device__ int slab_classify(double a, double b, double c, float2* bc, int mode) {
  if (a == 0.0 && b == 0.0) {
    if (c >= 0.0) return kNone;          // no constraint (e.g. outer == inner)
    *bc = make_float2(0.f, INFINITY);     // unsatisfiable: x' >= +inf (or y')
    return mode == kPreferY ? kYlo : kXlo;
  }
  constexpr double kSteep = static_cast<double>(1ull << VPIPG_SLAB_STEEP);
  const bool xform = mode == kMixed    ? fabs(a) >= fabs(b)
                     : mode == kPreferY ? fabs(a) > fabs(b) * kSteep
                                        : fabs(b) <= fabs(a) * kSteep;
  if (xform) {
    *bc = make_float2(static_cast<float>(-b / a), static_cast<float>(-c / a));
    return a > 0.0 ? kXlo : kXhi;
  }
  *bc = make_float2(static_cast<float>(-a / b), static_cast<float>(-c / b));
  return b > 0.0 ? kYlo : kYhi;
}

__device__ __forceinline__ uint32_t even_len(uint32_t c) { return (c + 1u) & ~1u; }

// Block-wide deterministic scatter of per-edge (class, coef) into the four
// groups of one slab table, each padded with neutral entries to an even
// length, and to at least one pair unless both groups of its side are empty
// (single-section table). Edge order is preserved inside a group.
__device__ void slab_scatter(int n, int (*cls_of)(int, const void*, float2*, int), const void* ctx,
                             float2* out, uint32_t* cnt_out) {
  __shared__ uint32_t s_base[kGroups];
  __shared__ uint32_t s_warp[kGroups][kPrepThreads / 32];
  __shared__ uint32_t s_count[3][kGroups];
  __shared__ int s_mode;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid < 3 * kGroups) s_count[tid / kGroups][tid % kGroups] = 0;
  __syncthreads();
  // pass 1: group sizes under each orientation mode
  for (int k = tid; k < n; k += kPrepThreads) {
    float2 bc;
    for (int m = 0; m < 3; ++m) {
      const int c = cls_of(k, ctx, &bc, m);
      if (c >= 0) atomicAdd(&s_count[m][c], 1u);
    }
  }
  __syncthreads();
  if (tid == 0) {
    // single-section candidates, cost = padded edges per point (ties: balance)
    int mode = kMixed;
    uint32_t best = UINT32_MAX;
    for (int m = kPreferY; m <= kPreferX; ++m) {
      const uint32_t* c = s_count[m];
      const bool single = m == kPreferY ? (c[kXlo] | c[kXhi]) == 0 : (c[kYlo] | c[kYhi]) == 0;
      const uint32_t lo = m == kPreferY ? c[kYlo] : c[kXlo];
      const uint32_t hi = m == kPreferY ? c[kYhi] : c[kXhi];
      const uint32_t plo = max(even_len(lo), 2u), phi = max(even_len(hi), 2u);
      const uint32_t cost = 4u * (plo + phi) + (plo > phi ? plo - phi : phi - plo);
      if (single && cost < best) {
        best = cost;
        mode = m;
      }
    }
    s_mode = mode;
    const uint32_t* cnt = s_count[mode];
    const bool x_empty = (cnt[kXlo] | cnt[kXhi]) == 0;
    const bool y_empty = (cnt[kYlo] | cnt[kYhi]) == 0;
    uint32_t acc = 0;
    for (int g = 0; g < kGroups; ++g) {
      s_base[g] = acc;
      // even length (two edges per 16-byte load) and at least one pair, so
      // the kernels can seed their running max / min from the first pair --
      // except that an empty side stays empty (single-section table)
      uint32_t padded = even_len(cnt[g]);
      const bool side_empty = g <= kXhi ? x_empty && !y_empty : y_empty;
      if (padded == 0 && !side_empty) padded = 2;
      cnt_out[g] = padded;
      for (uint32_t q = cnt[g]; q < padded; ++q)  // neutral pad entries
        out[acc + q] = make_float2(0.f, (g == kXlo || g == kYlo) ? -INFINITY : INFINITY);
      acc += padded;
    }
  }
  __syncthreads();
  const int mode = s_mode;
  // pass 2: ordered placement, one 256-edge chunk at a time
  for (int k0 = 0; k0 < n; k0 += kPrepThreads) {
    const int k = k0 + tid;
    float2 bc = make_float2(0.f, 0.f);
    const int c = (k < n) ? cls_of(k, ctx, &bc, mode) : kNone;
    uint32_t rank = 0;  // this edge's rank inside its group, within the warp
#pragma unroll
    for (int g = 0; g < kGroups; ++g) {
      const unsigned bal = __ballot_sync(0xffffffffu, c == g);
      if (c == g) rank = __popc(bal & ((1u << lane) - 1u));
      if (lane == 0) s_warp[g][warp] = __popc(bal);
    }
    __syncthreads();
    if (c >= 0) {
      uint32_t before = 0;
      for (int w = 0; w < warp; ++w) before += s_warp[c][w];
      out[s_base[c] + before + rank] = bc;
    }
    __syncthreads();
    if (tid < kGroups) {
      uint32_t tot = 0;
      for (int w = 0; w < kPrepThreads / 32; ++w) tot += s_warp[tid][w];
      s_base[tid] += tot;
    }
    __syncthreads();
  }
}

struct VorCtx {
  const double2* outer;
  double p0x, p0y, ox, oy;
};

// Voronoi half-plane k: |x - p0|^2 <= |x - pk|^2  <=>  d.(m - x) >= 0 with
// d = pk - p0 and m the midpoint (the perpendicular bisector, Eq. 9).
__device__ int vor_class(int k, const void* ctx, float2* bc, int mode) {
  const VorCtx& v = *static_cast<const VorCtx*>(ctx);
  const double2 pk = v.outer[k];
  const double dx = pk.x - v.p0x, dy = pk.y - v.p0y;
  const double mx = 0.5 * ((v.p0x - v.ox) + (pk.x - v.ox));
  const double my = 0.5 * ((v.p0y - v.oy) + (pk.y - v.oy));
  return slab_classify(-dx, -dy, dx * mx + dy * my, bc, mode);
}

struct OffCtx {
  const double* vx;
  const double* vy;
  int n;
  double ox, oy;
};

// Sign-of-offset edge e (j = e-1 -> i = e): inside iff lhs >= rhs, i.e.
// (q - v_j) x dv >= 0 (engines.cpp:150-152 with the flags == 0 branch).
__device__ int off_class(int e, const void* ctx, float2* bc, int mode) {
  const OffCtx& o = *static_cast<const OffCtx*>(ctx);
  const int i = e, j = (e + o.n - 1) % o.n;
  const double dvx = o.vx[i] - o.vx[j], dvy = o.vy[i] - o.vy[j];
  const double wx = o.vx[j] - o.ox, wy = o.vy[j] - o.oy;
  return slab_classify(-dvy, dvx, wx * dvy - wy * dvx, bc, mode);
}

// kInline: the input vertices / generators travel in the kernel's parameter
// bank (small polygons: no upload call); offsets in doubles, -1 = absent
template <bool kInline>
__global__ void __launch_bounds__(kPrepThreads) prep_kernel(const PrepArgs a0,
                                                            const __grid_constant__ PrepInline in) {
  __shared__ double s_inner[2];
  __shared__ int s_fail;  // min over failing edges of (edge * 8 + code): the first throw wins
  PrepArgs a = a0;
  if constexpr (kInline) {
    a.vv = in.vv_at >= 0 ? in.v + in.vv_at : nullptr;
    a.vr = in.vr_at >= 0 ? in.v + in.vr_at : nullptr;
    a.gen_in = in.gen_at >= 0 ? in.v + in.gen_at : nullptr;
  }
  const int tid = threadIdx.x;
  const int n = static_cast<int>(a.n);
  if (tid < 2 * kGroups) a.meta->cnt[tid / kGroups][tid % kGroups] = 0;  // kinds not prepared
  if (tid == 0) {
    s_fail = INT_MAX;
    double cx = 0.0, cy = 0.0;
    if (a.gen_in != nullptr) {  // explicit generator set
      cx = a.gen_in[0];
      cy = a.gen_in[1];
    } else if (a.vv != nullptr) {
      // centroid, geometry.cpp:106-120, sequential in the reference order
      const double* vv = a.vv;
      centroid_exact([vv, n](int k) { return make_double2(vv[k], vv[n + k]); }, n, &cx, &cy);
    } else if (a.vr != nullptr && n > 0) {  // crossing only: vertex mean as frame origin
      for (int i = 0; i < n; ++i) {
        cx += a.vr[i];
        cy += a.vr[n + i];
      }
      cx /= n;
      cy /= n;
    }
    s_inner[0] = cx;
    s_inner[1] = cy;
    // The fp32 tables live in the polygon-local frame:
    // origin = the centroid rounded to f32 (+0.0 for a zero coordinate, so
    // x - ox keeps every point bit for bit there); the test kernels subtract
    // it from each point, exactly for the points near the polygon (Sterbenz),
    // so a small polygon far from the origin keeps errors ~2^-24 of its extent
#ifndef VPIPG_LOCAL_FRAME
#define VPIPG_LOCAL_FRAME 1
#endif
    // A polygon whose centroid lies within its own extent of the origin keeps
    // the absolute frame (origin (0, 0): the kernels then skip the shift),
    // as accurate there since |x| <= ~2 extent for every point near it.
    const double* vsrc = a.vv ? a.vv : a.vr;
    double lo_x = INFINITY, hi_x = -INFINITY, lo_y = INFINITY, hi_y = -INFINITY;
    for (int i = 0; vsrc && i < n; ++i) {
      lo_x = fmin(lo_x, vsrc[i]);
      hi_x = fmax(hi_x, vsrc[i]);
      lo_y = fmin(lo_y, vsrc[n + i]);
      hi_y = fmax(hi_y, vsrc[n + i]);
    }
    const double extent = fmax(hi_x - lo_x, hi_y - lo_y);
    const bool local = VPIPG_LOCAL_FRAME && !(fmax(fabs(cx), fabs(cy)) <= extent);
    const float ox = local ? static_cast<float>(cx) + 0.f : 0.f;
    const float oy = local ? static_cast<float>(cy) + 0.f : 0.f;
    a.meta->inner_x = cx;
    a.meta->inner_y = cy;
    a.meta->ox = ox;
    a.meta->oy = oy;
  }
  __syncthreads();
  const double p0x = s_inner[0], p0y = s_inner[1];
  const double ox = static_cast<double>(a.meta->ox), oy = static_cast<double>(a.meta->oy);

  // ---- Voronoi generators (voronoi.cpp:60-71) ----
  if (a.kinds & kKindVoronoi) {
    if (a.gen_in != nullptr) {
      for (int k = tid; k < n; k += kPrepThreads)
        a.outer[k] = make_double2(a.gen_in[2 + 2 * k], a.gen_in[3 + 2 * k]);
    } else {
      for (int k = tid; k < n; k += kPrepThreads) {
        const int k1 = (k + 1) % n;
        // edge_coefficients + reflect_generator (voronoi.cpp:23-58, Eq. 8 fused)
        double2 g;
        const int rc = reflect_exact(make_double2(a.vv[k], a.vv[n + k]),
                                     make_double2(a.vv[k1], a.vv[n + k1]), p0x, p0y, &g);
        if (rc) {
          atomicMin(&s_fail, k * 8 + rc);  // DegenerateEdge / GeneratorCollision
          continue;
        }
        a.outer[k] = g;
      }
    }
    __syncthreads();
    VorCtx vc{a.outer, p0x, p0y, ox, oy};
    slab_scatter(n, vor_class, &vc, a.slab_coef[0], a.meta->cnt[0]);
  }

  // ---- sign-of-offset (engines.cpp:146-149) ----
  if (a.kinds & kKindOffset) {
    for (int e = tid; e < n; e += kPrepThreads) {
      const int i = e, j = (e + n - 1) % n;
      const double dvx = dsub(a.vv[i], a.vv[j]);
      const double dvy = dsub(a.vv[n + i], a.vv[n + j]);
      const double rhs = dsub(dmul(a.vv[n + j], dvx), dmul(a.vv[j], dvy));
      a.off[e] = OffsetEdgeF64{dvx, dvy, rhs, 0.0};
    }
    __syncthreads();
    OffCtx oc{a.vv, a.vv + n, n, ox, oy};
    slab_scatter(n, off_class, &oc, a.slab_coef[1], a.meta->cnt[1]);
  }

  // ---- ray crossing (engines.cpp:176-186), raw vertices ----
  if (a.kinds & kKindCrossing) {
    for (int e = tid; e < n; e += kPrepThreads) {
      const int i = e, j = (e + n - 1) % n;
      const double wx = a.vr[j], wy = a.vr[n + j], ux = a.vr[i], uy = a.vr[n + i];
      const double dvx = dsub(ux, wx), dvy = dsub(uy, wy);
      RayEdgeF64 r;
      r.wy = wy;
      r.uy = uy;
      r.dvx = dvx;
      r.dvy = dvy;
      r.rhs = dsub(dmul(wy, dvx), dmul(wx, dvy));
      r.min_x = smin(wx, ux);
      r.max_x = smax(wx, ux);
      r.min_y = smin(wy, uy);
      r.max_y = smax(wy, uy);
      r.going_up = uy > wy;
      r.pad_ = 0;
      a.ray[e] = r;
      // fp32 crossing record for vertex i (edge j -> i)
      // (u.x, u.y, dvx/dvy, w.x) in the local frame; w.x is rounded exactly
      // as vertex j's own .x, so either loop form of the kernel sees the
      // same g for a vertex
      const float bk = (dvy != 0.0) ? static_cast<float>(dvx / dvy) : 0.f;
      a.cross_vert[i] = make_float4(static_cast<float>(ux - ox), static_cast<float>(uy - oy), bk,
                                    static_cast<float>(wx - ox));
    }
  }
  // ---- band metric lines: edge k (v[k] -> v[k+1]) of the validated vertices,
  // else the raw ones, else the generator bisectors (voronoi.cpp:23-35, 73-82)
  {
    const double* vv = a.vv ? a.vv : a.vr;
    for (int k = tid; k < n; k += kPrepThreads) {
      double la, lb, lc;
      if (vv) {
        const int k1 = (k + 1) % n;
        la = vv[n + k] - vv[n + k1];
        lb = vv[k1] - vv[k];
        lc = -(la * vv[k] + lb * vv[n + k]);
      } else {  // bisector of p0 and outer[k]
        const double2 g = a.outer[k];
        la = g.x - p0x;
        lb = g.y - p0y;
        lc = -(la * 0.5 * (p0x + g.x) + lb * 0.5 * (p0y + g.y));
      }
      const double h = hypot(la, lb);
      const double s = h > 0.0 ? 1.0 / h : 0.0;
      a.lines[k] = make_double4(la * s, lb * s, lc * s, 0.0);
    }
  }
  __syncthreads();
  if (tid == 0) a.meta->status = (s_fail == INT_MAX) ? 0 : (s_fail & 7);
  if (a.host_out) {  // straight into the caller's mapped pinned block
    __syncthreads();
    const uint32_t* mw = reinterpret_cast<const uint32_t*>(a.meta);
    uint32_t* hm = reinterpret_cast<uint32_t*>(a.host_out);
    for (int i = tid; i < static_cast<int>(sizeof(PrepMeta) / 4); i += kPrepThreads) hm[i] = mw[i];
    if (a.tables_out) {
      for (int e = 0; e < 2; ++e) {
        float2* h = reinterpret_cast<float2*>(a.host_out + a.out_slab[e]);
        for (int i = tid; i < n + 4; i += kPrepThreads) h[i] = a.slab_coef[e][i];
      }
      float4* hc = reinterpret_cast<float4*>(a.host_out + a.out_cross);
      for (int i = tid; i < n; i += kPrepThreads) hc[i] = a.cross_vert[i];
    }
  }
}

}  // namespace

cudaError_t launch_prep(const PrepArgs& args, const PrepInline* in, cudaStream_t stream) {
  if (in) {
    prep_kernel<true><<<1, kPrepThreads, 0, stream>>>(args, *in);
  } else {
    static const PrepInline none{};
    prep_kernel<false><<<1, kPrepThreads, 0, stream>>>(args, none);
  }
  return cudaGetLastError();
}

}  // namespace vpipg
