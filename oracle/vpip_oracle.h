/*
 * vpip_oracle.h -- CPU restatement of the reference point-inclusion path.
 *
 * TEST INFRASTRUCTURE ONLY. This oracle is the checker for the B200 engine:
 * only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * load it. The product path (paper_2007_15385_b200/) never links or calls it.
 *
 * Every function restates the reference algorithm (arxiv 2007.15385, the
 * `vpip` C++ library under proj/) in plain C, with the same operation order,
 * so that compiled with -ffp-contract=off it produces the same bits as the
 * reference. Citations are to /root/reference/proj/... file:line.
 *
 * Parity pin: tests/test_oracle_golden.py checks this restatement against
 * the reference's own known-answer tests and against fixtures produced by the
 * reference itself (oracle/_ref, built from the reference sources by
 * oracle/Makefile; fixtures in tests/golden/, script tests/golden/make_golden.py).
 */
#ifndef VPIP_ORACLE_H
#define VPIP_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Error codes: 0 = ok, 1..7 = vpip::ErrorCode in declaration order
 * (proj/include/vpip/error.hpp:23-31). */
enum {
  VO_OK = 0,
  VO_TOO_FEW_VERTICES = 1,
  VO_NOT_CONVEX = 2,
  VO_DEGENERATE_EDGE = 3,
  VO_NON_FINITE = 4,
  VO_GENERATOR_COLLISION = 5,
  VO_INVALID_PARAMETER = 6,
  VO_PARSE_ERROR = 7
};

/* --- seeded sampling (proj/src/sampling.cpp) --- */
uint64_t vo_mix_seed(uint64_t seed, uint64_t salt);                  /* sampling.cpp:107-112 */
double vo_unit_from_u64(uint64_t r);                                 /* sampling.cpp:31-33 */
int vo_sample_points(size_t count, double min_x, double min_y, double max_x, double max_y,
                     uint64_t seed, double* xs, double* ys);         /* sampling.cpp:90-105 */
/* Regular n-gon (already validated: CCW by construction). sampling.cpp:50-61 */
int vo_regular_polygon(size_t n, double r, double cx, double cy, double* vx, double* vy);
/* Random strictly convex n-gon, validated. sampling.cpp:63-88 */
int vo_random_convex_polygon(size_t n, uint64_t seed, double r, double cx, double cy,
                             double* vx, double* vy);

/* --- geometry (proj/src/geometry.cpp) --- */
/* In-place validation: checks, reverses to CCW if needed. geometry.cpp:53-98 */
int vo_validate_polygon(double* vx, double* vy, size_t n, double convexity_eps, int* reversed);
double vo_signed_area(const double* vx, const double* vy, size_t n);  /* geometry.cpp:100-104 */
void vo_centroid(const double* vx, const double* vy, size_t n, double* cx, double* cy); /* :106-120 */
void vo_bounding_box(const double* vx, const double* vy, size_t n, double box[4]);     /* :39-51 */
void vo_box_scaled(const double box[4], double factor, double out[4]); /* geometry.hpp:64-69 */

/* --- voronoi conversion (proj/src/voronoi.cpp) --- */
int vo_edge_coefficients(double qix, double qiy, double qjx, double qjy, double abc[3]); /* :23-31 */
int vo_reflect_generator(double px, double py, const double abc[3], double* rx, double* ry); /* :46-58 */
void vo_foot_of_perpendicular(double px, double py, const double abc[3], double* fx, double* fy); /* :37-44 */
/* inner = centroid, outer[k] = reflect(inner, edge k). voronoi.cpp:60-71 */
int vo_to_voronoi(const double* vx, const double* vy, size_t n, double* inner_xy, double* outer_xy);
double vo_edge_line_distance(const double* vx, const double* vy, size_t n, double px, double py); /* :73-82 */

/* --- batch engines (proj/src/engines.cpp); byte masks, 1 = inside --- */
void vo_voronoi_batch(const double* inner_xy, const double* outer_xy, size_t n,
                      const double* xs, const double* ys, size_t m, uint8_t* out);    /* :65-104 */
void vo_offset_batch(const double* vx, const double* vy, size_t n,
                     const double* xs, const double* ys, size_t m, uint8_t* out);     /* :136-160 */
void vo_ray_batch(const double* vx, const double* vy, size_t n,
                  const double* xs, const double* ys, size_t m, uint8_t* out);        /* :165-204 */
/* Scalar early-exit variants. engines.cpp:235-241, :304-318, :331-350, :352-367 */
int vo_voronoi_contains(const double* inner_xy, const double* outer_xy, size_t n, double px, double py);
int vo_offset_contains(const double* vx, const double* vy, size_t n, double px, double py);
int vo_ray_contains(const double* vx, const double* vy, size_t n, double px, double py);
int vo_ray_count(const double* vx, const double* vy, size_t n, double px, double py);
uint64_t vo_count_inside(const uint8_t* mask, size_t m);                              /* :215-217 */

/* PIPM payload: bit j of the byte stream is point j, LSB-first. io.cpp:272-279 */
void vo_pack_mask_lsb(const uint8_t* mask, size_t m, uint8_t* bytes);

/* Counter-based point stream used for configs whose batches are too large to
 * pre-sample on the host: point j = (lo_x + w*U(mix_seed(seed, 2j)),
 * lo_y + h*U(mix_seed(seed, 2j+1))), rounded to float32 and widened back.
 * U is the reference's top-53-bit uniform (sampling.cpp:31-33). The device
 * generator in the product produces the same float32 values. */
void vo_counter_points_f32(uint64_t seed, uint64_t first, size_t count, double min_x,
                           double min_y, double max_x, double max_y, float* xs, float* ys);

/* Polygon-database join (config 4). Pair generator restating the device
 * generator: id = floor(U(seed,3j) * npoly), point = c[id] + (2U-1) * r[id]. */
void vo_join_pairs_f32(uint64_t seed, uint64_t first, size_t m, uint32_t npoly, const double* cx,
                       const double* cy, const double* r, float* xs, float* ys, uint32_t* ids);
/* Per-polygon validate_polygon status (0 or ErrorCode + 1) of a CSR batch. */
void vo_csr_status(const uint32_t* offsets, const double* vx, const double* vy, uint32_t npoly,
                   int32_t* status);
/* Masks of one engine (0 voronoi, 1 offset, 2 crossing) for (point, id) pairs:
 * each pair is tested against its polygon exactly as the reference batch
 * kernels test one point (voronoi/offset on the validated polygon, crossing on
 * the raw vertices); pairs whose polygon failed validation (voronoi/offset)
 * or whose id is out of range are 0. Points are f64. */
void vo_join_masks(const uint32_t* offsets, const double* vx, const double* vy, uint32_t npoly,
                   int engine, const double* xs, const double* ys, const uint32_t* ids, size_t m,
                   uint8_t* out);

#ifdef __cplusplus
}
#endif
#endif
