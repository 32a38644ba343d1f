// exact_geom.cuh -- the reference's f64 geometry, operation for operation,
// shared by the device kernels (prep.cu, csr.cu) and the host code (capi.cu,
// vpip_api.cpp): ONE definition of each check and of the seed mixer.
//
// Every expression below is the reference's (-ffp-contract=off) expression:
// on the device written with explicitly rounded intrinsics, which nvcc never
// fuses into FMAs; on the host plain operators in translation units compiled
// with -ffp-contract=off, as the reference is. Results are bit-identical to
// the reference build:
//   centroid           geometry.cpp:106-120
//   edge_coefficients  voronoi.cpp:23-31
//   reflect_generator  voronoi.cpp:46-58 (the fused mirror of PAPER.md Eq. 8)
//   validate_polygon   geometry.cpp:53-98 (checks, order, CCW normalisation)
//   mix_seed           sampling.cpp:107-112 (SplitMix64 finaliser)
#pragma once

#include <cmath>
#include <cstdint>

#include <vector_functions.h>
#include <vector_types.h>

#if defined(__CUDACC__)
#define VPIPG_HD __host__ __device__ __forceinline__
#else
#define VPIPG_HD inline
#endif

namespace vpipg {

#if defined(__CUDA_ARCH__)
VPIPG_HD double dmul(double a, double b) { return __dmul_rn(a, b); }
VPIPG_HD double dadd(double a, double b) { return __dadd_rn(a, b); }
VPIPG_HD double dsub(double a, double b) { return __dsub_rn(a, b); }
VPIPG_HD double ddiv(double a, double b) { return __ddiv_rn(a, b); }
VPIPG_HD bool dfinite(double a) { return isfinite(a); }
VPIPG_HD double datan2(double y, double x) { return atan2(y, x); }
#else
VPIPG_HD double dmul(double a, double b) { return a * b; }
VPIPG_HD double dadd(double a, double b) { return a + b; }
VPIPG_HD double dsub(double a, double b) { return a - b; }
VPIPG_HD double ddiv(double a, double b) { return a / b; }
VPIPG_HD bool dfinite(double a) { return std::isfinite(a); }
VPIPG_HD double datan2(double y, double x) { return std::atan2(y, x); }
#endif
// std::min / std::max semantics (engines.cpp:183-186)
VPIPG_HD double smin(double a, double b) { return (b < a) ? b : a; }
VPIPG_HD double smax(double a, double b) { return (a < b) ? b : a; }

// mix_seed (sampling.cpp:107-112): the device point streams (fill.cu,
// csr.cu) and the host samplers (vpip_api.cpp) draw from this one definition
VPIPG_HD uint64_t mix_seed(uint64_t seed, uint64_t salt) {
  uint64_t z = seed + 0x9e3779b97f4a7c15ULL * (salt + 1);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

// Vertex accessor: V(k) -> (x, y) of vertex k of an n-gon.
template <class V>
VPIPG_HD void centroid_exact(const V& v, int n, double* cx, double* cy) {
  double area2 = 0.0, sx = 0.0, sy = 0.0;
  for (int i = 0, j = n - 1; i < n; j = i++) {
    const double2 a = v(j), b = v(i);
    const double d = dsub(dmul(a.x, b.y), dmul(b.x, a.y));
    area2 = dadd(area2, d);
    sx = dadd(sx, dmul(dadd(a.x, b.x), d));
    sy = dadd(sy, dmul(dadd(a.y, b.y), d));
  }
  *cx = ddiv(sx, dmul(3.0, area2));
  *cy = ddiv(sy, dmul(3.0, area2));
}

// Mirror of p across the line through edge (qi, qj). Returns 0, 3
// (DegenerateEdge) or 5 (GeneratorCollision), the reference's throw sites.
VPIPG_HD int reflect_exact(double2 qi, double2 qj, double px, double py,
                                             double2* out) {
  const double ea = dsub(qi.y, qj.y);
  const double eb = dsub(qj.x, qi.x);
  const double ec = -dadd(dmul(ea, qi.x), dmul(eb, qi.y));
  const double denom = dadd(dmul(ea, ea), dmul(eb, eb));
  if (denom <= 1e-24) return 3;
  if (fabs(dadd(dadd(dmul(ea, px), dmul(eb, py)), ec)) <= dmul(1e-12, denom)) return 5;
  const double t1 = dmul(dsub(dmul(eb, eb), dmul(ea, ea)), px);
  const double t2 = dmul(dmul(dmul(2.0, ea), eb), py);
  const double t3 = dmul(dmul(2.0, ec), ea);
  const double u1 = dmul(dmul(dmul(-2.0, ea), eb), px);
  const double u2 = dmul(dsub(dmul(ea, ea), dmul(eb, eb)), py);
  const double u3 = dmul(dmul(2.0, ec), eb);
  *out = make_double2(ddiv(dsub(dsub(t1, t2), t3), denom), ddiv(dsub(dadd(u1, u2), u3), denom));
  return 0;
}

// validate_polygon without the exception: 0 or ErrorCode + 1, and whether
// the vertex order must be reversed to make it counter-clockwise. `at` (may
// be null) receives the offending vertex (NonFinite, NotConvex: the index in
// the CCW order) or edge end i of edge j -> i (DegenerateEdge), -1 when the
// whole polygon is at fault, for the reference's error messages.
template <class V>
VPIPG_HD int validate_exact(const V& v, int n, bool* reversed, double convexity_eps = 1e-12,
                            int* at = nullptr) {
  *reversed = false;
  int where = -1;
  if (!at) at = &where;
  *at = -1;
  for (int k = 0; k < n; ++k) {
    const double2 p = v(k);
    if (!dfinite(p.x) || !dfinite(p.y)) {
      *at = k;
      return 4;  // NonFinite
    }
  }
  if (n < 3) return 1;  // TooFewVertices
  for (int i = 0, j = n - 1; i < n; j = i++) {
    const double2 a = v(j), b = v(i);
    const double dx = dsub(a.x, b.x), dy = dsub(a.y, b.y);
    if (dadd(dmul(dx, dx), dmul(dy, dy)) <= 1e-24) {
      *at = i;
      return 3;  // DegenerateEdge
    }
  }
  double sum = 0.0;
  for (int i = 0, j = n - 1; i < n; j = i++) {
    const double2 a = v(j), b = v(i);
    sum = dadd(sum, dsub(dmul(a.x, b.y), dmul(b.x, a.y)));
  }
  *reversed = sum < 0.0;
  const bool rev = *reversed;
  auto w = [&](int k) { return v(rev ? n - 1 - k : k); };
  double total_turn = 0.0;
  for (int i = 0; i < n; ++i) {
    const double2 prev = w((i + n - 1) % n), cur = w(i), next = w((i + 1) % n);
    const double inx = dsub(cur.x, prev.x), iny = dsub(cur.y, prev.y);
    const double outx = dsub(next.x, cur.x), outy = dsub(next.y, cur.y);
    const double cr = dsub(dmul(inx, outy), dmul(iny, outx));
    if (cr <= convexity_eps) {
      *at = i;
      return 2;  // NotConvex (collinear or reflex)
    }
    total_turn = dadd(total_turn, datan2(cr, dadd(dmul(inx, outx), dmul(iny, outy))));
  }
  if (total_turn >= dmul(3.0, 3.141592653589793)) return 2;  // winds more than once
  return 0;
}

}  // namespace vpipg
