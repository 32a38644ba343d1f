/*
 * vpip_oracle.c -- CPU restatement of the reference point-inclusion path.
 *
 * TEST INFRASTRUCTURE ONLY (see vpip_oracle.h). Compile with
 * -ffp-contract=off (oracle/Makefile does): the reference's Release build
 * uses -ffp-contract=off (proj/CMakeLists.txt:13-17), so no FMA contraction
 * may change the bits of any expression below. Expression shapes follow the
 * reference exactly; C evaluates a*b*c as (a*b)*c like C++ does.
 */
#include "vpip_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------ */
/* std::mt19937_64, restated from its published definition (Matsumoto and
 * Nishimura 2000; C++11 [rand.predef]: w=64 n=312 m=156 r=31
 * a=0xb5026f5aa96619e9 u=29 d=0x5555555555555555 s=17 b=0x71d67fffeda60000
 * t=37 c=0xfff7eee000000000 l=43 f=6364136223846793005). The reference seeds
 * it with the 64-bit seed directly (sampling.cpp:72, :96). */
typedef struct {
  uint64_t mt[312];
  int idx;
} mt64;

static void mt64_seed(mt64* g, uint64_t seed) {
  g->mt[0] = seed;
  for (int i = 1; i < 312; ++i)
    g->mt[i] = 6364136223846793005ULL * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) + (uint64_t)i;
  g->idx = 312;
}

static uint64_t mt64_next(mt64* g) {
  static const uint64_t kUpper = 0xFFFFFFFF80000000ULL, kLower = 0x7FFFFFFFULL;
  if (g->idx >= 312) {
    for (int i = 0; i < 312; ++i) {
      uint64_t x = (g->mt[i] & kUpper) | (g->mt[(i + 1) % 312] & kLower);
      uint64_t xa = x >> 1;
      if (x & 1ULL) xa ^= 0xB5026F5AA96619E9ULL;
      g->mt[i] = g->mt[(i + 156) % 312] ^ xa;
    }
    g->idx = 0;
  }
  uint64_t y = g->mt[g->idx++];
  y ^= (y >> 29) & 0x5555555555555555ULL;
  y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
  y ^= (y << 37) & 0xFFF7EEE000000000ULL;
  y ^= y >> 43;
  return y;
}

/* sampling.cpp:31-33: top 53 bits scaled by 2^-53. */
double vo_unit_from_u64(uint64_t r) { return (double)(r >> 11) * 0x1.0p-53; }

static double unit_real(mt64* g) { return vo_unit_from_u64(mt64_next(g)); }

/* sampling.cpp:107-112 (splitmix64 finaliser). */
uint64_t vo_mix_seed(uint64_t seed, uint64_t salt) {
  uint64_t z = seed + 0x9e3779b97f4a7c15ULL * (salt + 1);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

/* std::min / std::max semantics: min(a, b) = (b < a) ? b : a. */
static inline double smin(double a, double b) { return (b < a) ? b : a; }
static inline double smax(double a, double b) { return (a < b) ? b : a; }

static const double kPi = 3.141592653589793238462643383279502884;

/* sampling.cpp:90-105 */
int vo_sample_points(size_t count, double min_x, double min_y, double max_x, double max_y,
                     uint64_t seed, double* xs, double* ys) {
  if (!(isfinite(min_x) && isfinite(min_y) && isfinite(max_x) && isfinite(max_y) &&
        min_x < max_x && min_y < max_y))
    return VO_INVALID_PARAMETER;
  mt64 g;
  mt64_seed(&g, seed);
  const double w = max_x - min_x;
  const double h = max_y - min_y;
  for (size_t j = 0; j < count; ++j) {
    xs[j] = min_x + w * unit_real(&g);
    ys[j] = min_y + h * unit_real(&g);
  }
  return VO_OK;
}

static int check_polygon_params(size_t n, double r, double cx, double cy) {
  if (n < 3) return VO_INVALID_PARAMETER;
  if (!isfinite(r) || r <= 0.0) return VO_INVALID_PARAMETER;
  if (!isfinite(cx) || !isfinite(cy)) return VO_INVALID_PARAMETER;
  return VO_OK;
}

/* sampling.cpp:50-61; validate_polygon keeps the CCW order it produces. */
int vo_regular_polygon(size_t n, double r, double cx, double cy, double* vx, double* vy) {
  int rc = check_polygon_params(n, r, cx, cy);
  if (rc) return rc;
  for (size_t k = 0; k < n; ++k) {
    const double angle = 2.0 * kPi * (double)k / (double)n + kPi / 2.0;
    vx[k] = cx + r * cos(angle);
    vy[k] = cy + r * sin(angle);
  }
  int rev = 0;
  return vo_validate_polygon(vx, vy, n, 1e-12, &rev);
}

static int cmp_double(const void* a, const void* b) {
  const double x = *(const double*)a, y = *(const double*)b;
  return (x > y) - (x < y);
}

/* sampling.cpp:63-88 */
int vo_random_convex_polygon(size_t n, uint64_t seed, double r, double cx, double cy,
                             double* vx, double* vy) {
  int rc = check_polygon_params(n, r, cx, cy);
  if (rc) return rc;
  mt64 g;
  mt64_seed(&g, seed);
  const double min_gap = 2.0 * kPi / (20.0 * (double)n);
  double* angles = (double*)malloc(n * sizeof(double));
  if (!angles) return VO_INVALID_PARAMETER;
  for (int attempt = 0; attempt < 1024; ++attempt) {
    for (size_t k = 0; k < n; ++k) angles[k] = 2.0 * kPi * unit_real(&g);
    qsort(angles, n, sizeof(double), cmp_double);
    int spaced = angles[0] + 2.0 * kPi - angles[n - 1] >= min_gap;
    for (size_t k = 1; spaced && k < n; ++k) spaced = angles[k] - angles[k - 1] >= min_gap;
    if (!spaced) continue;
    for (size_t k = 0; k < n; ++k) {
      vx[k] = cx + r * cos(angles[k]);
      vy[k] = cy + r * sin(angles[k]);
    }
    free(angles);
    int rev = 0;
    return vo_validate_polygon(vx, vy, n, 1e-12, &rev);
  }
  free(angles);
  return VO_INVALID_PARAMETER;
}

/* geometry.cpp:28-35: twice the signed area, cyclic pairs (j, i) = (n-1, 0), (0, 1), ... */
static double shoelace_sum(const double* vx, const double* vy, size_t n) {
  double sum = 0.0;
  for (size_t i = 0, j = n - 1; i < n; j = i++) sum += vx[j] * vy[i] - vx[i] * vy[j];
  return sum;
}

/* geometry.cpp:53-98 */
int vo_validate_polygon(double* vx, double* vy, size_t n, double convexity_eps, int* reversed) {
  for (size_t i = 0; i < n; ++i)
    if (!isfinite(vx[i]) || !isfinite(vy[i])) return VO_NON_FINITE;
  if (n < 3) return VO_TOO_FEW_VERTICES;
  for (size_t i = 0, j = n - 1; i < n; j = i++) {
    const double dx = vx[j] - vx[i];
    const double dy = vy[j] - vy[i];
    if (dx * dx + dy * dy <= 1e-24) return VO_DEGENERATE_EDGE;
  }
  *reversed = 0;
  if (shoelace_sum(vx, vy, n) < 0.0) {
    for (size_t a = 0, b = n - 1; a < b; ++a, --b) {
      double t = vx[a]; vx[a] = vx[b]; vx[b] = t;
      t = vy[a]; vy[a] = vy[b]; vy[b] = t;
    }
    *reversed = 1;
  }
  double total_turn = 0.0;
  for (size_t i = 0; i < n; ++i) {
    const size_t p = (i + n - 1) % n, q = (i + 1) % n;
    const double inx = vx[i] - vx[p], iny = vy[i] - vy[p];
    const double outx = vx[q] - vx[i], outy = vy[q] - vy[i];
    const double cr = inx * outy - iny * outx;
    if (cr <= convexity_eps) return VO_NOT_CONVEX;
    total_turn += atan2(cr, inx * outx + iny * outy);
  }
  if (total_turn >= 3.0 * kPi) return VO_NOT_CONVEX;
  return VO_OK;
}

double vo_signed_area(const double* vx, const double* vy, size_t n) {
  return 0.5 * shoelace_sum(vx, vy, n);
}

/* geometry.cpp:106-120 */
void vo_centroid(const double* vx, const double* vy, size_t n, double* cx, double* cy) {
  double area2 = 0.0, sx = 0.0, sy = 0.0;
  for (size_t i = 0, j = n - 1; i < n; j = i++) {
    const double d = vx[j] * vy[i] - vx[i] * vy[j];
    area2 += d;
    sx += (vx[j] + vx[i]) * d;
    sy += (vy[j] + vy[i]) * d;
  }
  *cx = sx / (3.0 * area2);
  *cy = sy / (3.0 * area2);
}

/* geometry.cpp:39-51 */
void vo_bounding_box(const double* vx, const double* vy, size_t n, double box[4]) {
  box[0] = vx[0]; box[1] = vy[0]; box[2] = vx[0]; box[3] = vy[0];
  for (size_t i = 0; i < n; ++i) {
    box[0] = smin(box[0], vx[i]);
    box[1] = smin(box[1], vy[i]);
    box[2] = smax(box[2], vx[i]);
    box[3] = smax(box[3], vy[i]);
  }
}

/* geometry.hpp:64-69: Box::scaled */
void vo_box_scaled(const double box[4], double factor, double out[4]) {
  const double cx = 0.5 * (box[0] + box[2]);
  const double cy = 0.5 * (box[1] + box[3]);
  const double hw = 0.5 * factor * (box[2] - box[0]);
  const double hh = 0.5 * factor * (box[3] - box[1]);
  out[0] = cx - hw; out[1] = cy - hh; out[2] = cx + hw; out[3] = cy + hh;
}

/* voronoi.cpp:23-31 */
int vo_edge_coefficients(double qix, double qiy, double qjx, double qjy, double abc[3]) {
  const double a = qiy - qjy;
  const double b = qjx - qix;
  const double c = -(a * qix + b * qiy);
  if (a * a + b * b <= 1e-24) return VO_DEGENERATE_EDGE;
  abc[0] = a; abc[1] = b; abc[2] = c;
  return VO_OK;
}

/* voronoi.cpp:37-44 */
void vo_foot_of_perpendicular(double px, double py, const double abc[3], double* fx, double* fy) {
  const double a = abc[0], b = abc[1], c = abc[2];
  const double denom = a * a + b * b;
  *fx = (b * b * px - a * b * py - c * a) / denom;
  *fy = (-a * b * px + a * a * py - c * b) / denom;
}

/* voronoi.cpp:46-58: the fused mirror of Eq. 8 */
int vo_reflect_generator(double px, double py, const double abc[3], double* rx, double* ry) {
  const double a = abc[0], b = abc[1], c = abc[2];
  const double denom = a * a + b * b;
  if (fabs(a * px + b * py + c) <= 1e-12 * denom) return VO_GENERATOR_COLLISION;
  *rx = ((b * b - a * a) * px - 2.0 * a * b * py - 2.0 * c * a) / denom;
  *ry = (-2.0 * a * b * px + (a * a - b * b) * py - 2.0 * c * b) / denom;
  return VO_OK;
}

/* voronoi.cpp:60-71 */
int vo_to_voronoi(const double* vx, const double* vy, size_t n, double* inner_xy, double* outer_xy) {
  vo_centroid(vx, vy, n, &inner_xy[0], &inner_xy[1]);
  for (size_t k = 0; k < n; ++k) {
    const size_t k1 = (k + 1) % n;
    double abc[3];
    int rc = vo_edge_coefficients(vx[k], vy[k], vx[k1], vy[k1], abc);
    if (rc) return rc;
    rc = vo_reflect_generator(inner_xy[0], inner_xy[1], abc, &outer_xy[2 * k], &outer_xy[2 * k + 1]);
    if (rc) return rc;
  }
  return VO_OK;
}

/* voronoi.cpp:33-35 and :73-82 */
double vo_edge_line_distance(const double* vx, const double* vy, size_t n, double px, double py) {
  double nearest = INFINITY;
  for (size_t k = 0; k < n; ++k) {
    const size_t k1 = (k + 1) % n;
    double abc[3];
    if (vo_edge_coefficients(vx[k], vy[k], vx[k1], vy[k1], abc)) return NAN;
    const double d = fabs(abc[0] * px + abc[1] * py + abc[2]) / hypot(abc[0], abc[1]);
    nearest = smin(nearest, d);
  }
  return nearest;
}

/* engines.cpp:65-104 (the per-point operation sequence; the reference's
 * 4096-point blocking only reorders which point is visited when). */
void vo_voronoi_batch(const double* inner_xy, const double* outer_xy, size_t n,
                      const double* xs, const double* ys, size_t m, uint8_t* out) {
  const double ix = inner_xy[0], iy = inner_xy[1];
  for (size_t j = 0; j < m; ++j) {
    const double dx = xs[j] - ix, dy = ys[j] - iy;
    const double inner_sq = dx * dx + dy * dy;
    uint8_t inside = 1;
    for (size_t k = 0; k < n; ++k) {
      const double ox = xs[j] - outer_xy[2 * k], oy = ys[j] - outer_xy[2 * k + 1];
      const double outer_sq = ox * ox + oy * oy;
      inside &= (uint8_t)(inner_sq <= outer_sq);
    }
    out[j] = inside;
  }
}

/* engines.cpp:136-160: flags counts strict right-of-edge tests; 0 or n = inside */
void vo_offset_batch(const double* vx, const double* vy, size_t n,
                     const double* xs, const double* ys, size_t m, uint8_t* out) {
  for (size_t q = 0; q < m; ++q) {
    uint32_t flags = 0;
    for (size_t i = 0, j = n - 1; i < n; j = i++) {
      const double dvx = vx[i] - vx[j];
      const double dvy = vy[i] - vy[j];
      const double rhs = vy[j] * dvx - vx[j] * dvy;
      const double lhs = ys[q] * dvx - xs[q] * dvy;
      flags += (uint32_t)(lhs < rhs);
    }
    out[q] = (uint8_t)((flags == 0u) | (flags == (uint32_t)n));
  }
}

/* engines.cpp:165-204 */
void vo_ray_batch(const double* vx, const double* vy, size_t n,
                  const double* xs, const double* ys, size_t m, uint8_t* out) {
  for (size_t q = 0; q < m; ++q) {
    const double qx = xs[q], qy = ys[q];
    uint8_t parity = 0, on_edge = 0;
    for (size_t i = 0, j = n - 1; i < n; j = i++) {
      const double wx = vx[j], wy = vy[j], ux = vx[i], uy = vy[i];
      const double dvx = ux - wx, dvy = uy - wy;
      const double rhs = wy * dvx - wx * dvy;
      const int going_up = uy > wy;
      const double min_x = smin(wx, ux), max_x = smax(wx, ux);
      const double min_y = smin(wy, uy), max_y = smax(wy, uy);
      const int in_range = (uy > qy) != (wy > qy);
      const double lhs = qy * dvx - qx * dvy;
      const int on_left = (lhs != rhs) & ((lhs > rhs) == going_up);
      parity ^= (uint8_t)(in_range & on_left);
      const int on_segment = (lhs == rhs) & (qx >= min_x) & (qx <= max_x) & (qy >= min_y) &
                             (qy <= max_y);
      on_edge |= (uint8_t)on_segment;
    }
    out[q] = (uint8_t)(on_edge | parity);
  }
}

/* engines.cpp:235-241 */
int vo_voronoi_contains(const double* inner_xy, const double* outer_xy, size_t n, double px,
                        double py) {
  const double dx = px - inner_xy[0], dy = py - inner_xy[1];
  const double inner_sq = dx * dx + dy * dy;
  for (size_t k = 0; k < n; ++k) {
    const double ox = px - outer_xy[2 * k], oy = py - outer_xy[2 * k + 1];
    if (ox * ox + oy * oy < inner_sq) return 0;
  }
  return 1;
}

/* engines.cpp:304-318 */
int vo_offset_contains(const double* vx, const double* vy, size_t n, double px, double py) {
  for (size_t i = 0, j = n - 1; i < n; j = i++) {
    const double dvx = vx[i] - vx[j], dvy = vy[i] - vy[j];
    const double lhs = py * dvx - px * dvy;
    const double rhs = vy[j] * dvx - vx[j] * dvy;
    if (lhs < rhs) return 0;
  }
  return 1;
}

/* engines.cpp:331-350 */
int vo_ray_contains(const double* vx, const double* vy, size_t n, double px, double py) {
  int crossings = 0;
  for (size_t i = 0, j = n - 1; i < n; j = i++) {
    const double wx = vx[j], wy = vy[j], ux = vx[i], uy = vy[i];
    const double dvx = ux - wx, dvy = uy - wy;
    const int in_range = (uy > py) != (wy > py);
    const double lhs = py * dvx - px * dvy;
    const double rhs = wy * dvx - wx * dvy;
    const int on_left = (lhs != rhs) && ((lhs > rhs) == (uy > wy));
    crossings += (in_range && on_left);
    if (lhs == rhs && px >= smin(wx, ux) && px <= smax(wx, ux) && py >= smin(wy, uy) &&
        py <= smax(wy, uy))
      return 1;
  }
  return (crossings & 1) != 0;
}

/* engines.cpp:352-367 */
int vo_ray_count(const double* vx, const double* vy, size_t n, double px, double py) {
  int crossings = 0;
  for (size_t i = 0, j = n - 1; i < n; j = i++) {
    const double wx = vx[j], wy = vy[j], ux = vx[i], uy = vy[i];
    const double dvx = ux - wx, dvy = uy - wy;
    const int in_range = (uy > py) != (wy > py);
    const double lhs = py * dvx - px * dvy;
    const double rhs = wy * dvx - wx * dvy;
    const int on_left = (lhs != rhs) && ((lhs > rhs) == (uy > wy));
    crossings += (in_range && on_left);
  }
  return crossings;
}

uint64_t vo_count_inside(const uint8_t* mask, size_t m) {
  uint64_t s = 0;
  for (size_t j = 0; j < m; ++j) s += mask[j];
  return s;
}

/* io.cpp:272-279: ceil(m/8) bytes, bit (j % 8) of byte j/8 is point j */
void vo_pack_mask_lsb(const uint8_t* mask, size_t m, uint8_t* bytes) {
  memset(bytes, 0, (m + 7) / 8);
  for (size_t j = 0; j < m; ++j)
    if (mask[j]) bytes[j / 8] |= (uint8_t)(1u << (j % 8));
}

void vo_counter_points_f32(uint64_t seed, uint64_t first, size_t count, double min_x,
                           double min_y, double max_x, double max_y, float* xs, float* ys) {
  const double w = max_x - min_x, h = max_y - min_y;
  for (size_t t = 0; t < count; ++t) {
    const uint64_t j = first + t;
    xs[t] = (float)(min_x + w * vo_unit_from_u64(vo_mix_seed(seed, 2 * j)));
    ys[t] = (float)(min_y + h * vo_unit_from_u64(vo_mix_seed(seed, 2 * j + 1)));
  }
}

/* ---- polygon-database join helpers (config 4) ---- */
void vo_join_pairs_f32(uint64_t seed, uint64_t first, size_t m, uint32_t npoly, const double* cx,
                       const double* cy, const double* r, float* xs, float* ys, uint32_t* ids) {
  for (size_t t = 0; t < m; ++t) {
    const uint64_t j = first + t;
    uint32_t id = (uint32_t)(vo_unit_from_u64(vo_mix_seed(seed, 3 * j)) * (double)npoly);
    if (id >= npoly) id = npoly - 1;
    const double ux = 2.0 * vo_unit_from_u64(vo_mix_seed(seed, 3 * j + 1)) - 1.0;
    const double uy = 2.0 * vo_unit_from_u64(vo_mix_seed(seed, 3 * j + 2)) - 1.0;
    xs[t] = (float)(cx[id] + ux * r[id]);
    ys[t] = (float)(cy[id] + uy * r[id]);
    ids[t] = id;
  }
}

void vo_csr_status(const uint32_t* offsets, const double* vx, const double* vy, uint32_t npoly,
                   int32_t* status) {
  for (uint32_t i = 0; i < npoly; ++i) {
    const size_t s = offsets[i], n = offsets[i + 1] - offsets[i];
    double* px = (double*)malloc((n ? n : 1) * sizeof(double));
    double* py = (double*)malloc((n ? n : 1) * sizeof(double));
    memcpy(px, vx + s, n * sizeof(double));
    memcpy(py, vy + s, n * sizeof(double));
    int rev = 0;
    status[i] = vo_validate_polygon(px, py, n, 1e-12, &rev);
    if (status[i] == 0) {
      double* outer = (double*)malloc(2 * n * sizeof(double));
      double inner[2];
      status[i] = vo_to_voronoi(px, py, n, inner, outer);
      free(outer);
    }
    free(px);
    free(py);
  }
}

void vo_join_masks(const uint32_t* offsets, const double* vx, const double* vy, uint32_t npoly,
                   int engine, const double* xs, const double* ys, const uint32_t* ids, size_t m,
                   uint8_t* out) {
  /* per polygon: validated vertices and generators, computed once */
  const size_t nv = offsets[npoly];
  double* cvx = (double*)malloc((nv ? nv : 1) * sizeof(double));
  double* cvy = (double*)malloc((nv ? nv : 1) * sizeof(double));
  double* outer = (double*)malloc((nv ? 2 * nv : 2) * sizeof(double));
  double* inner = (double*)malloc(2 * (npoly ? npoly : 1) * sizeof(double));
  int* ok = (int*)malloc((npoly ? npoly : 1) * sizeof(int));
  memcpy(cvx, vx, nv * sizeof(double));
  memcpy(cvy, vy, nv * sizeof(double));
  for (uint32_t i = 0; i < npoly; ++i) {
    const size_t s = offsets[i], n = offsets[i + 1] - offsets[i];
    int rev = 0;
    ok[i] = vo_validate_polygon(cvx + s, cvy + s, n, 1e-12, &rev) == 0;
    if (ok[i]) ok[i] = vo_to_voronoi(cvx + s, cvy + s, n, inner + 2 * i, outer + 2 * s) == 0;
  }
  for (size_t j = 0; j < m; ++j) {
    const uint32_t id = ids[j];
    uint8_t r = 0;
    if (id < npoly) {
      const size_t s = offsets[id], n = offsets[id + 1] - offsets[id];
      if (engine == 2) {
        vo_ray_batch(vx + s, vy + s, n, xs + j, ys + j, 1, &r);
      } else if (ok[id]) {
        if (engine == 0) vo_voronoi_batch(inner + 2 * id, outer + 2 * s, n, xs + j, ys + j, 1, &r);
        else vo_offset_batch(cvx + s, cvy + s, n, xs + j, ys + j, 1, &r);
      }
    }
    out[j] = r;
  }
  free(cvx); free(cvy); free(outer); free(inner); free(ok);
}
