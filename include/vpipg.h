/*
 * vpipg.h -- C-ABI of the B200 point-inclusion engine (libvpipg.so).
 *
 * This is the drop-in boundary for the reference's hot path (arxiv 2007.15385,
 * the `vpip` C++ library, /root/reference/proj). Each entry point names the
 * reference interface it replaces. The reference has no FFI of its own; its
 * callers are C++ (the CLI, the bench harness, the tests), so the binding a
 * maintainer adds is the C++ shim in include/vpip/ headers (same signatures as
 * proj/include/vpip/, implemented over this ABI), or a ctypes/cffi stub
 * from Python -- see INTEGRATION.md.
 *
 * Conventions
 *  - Return 0 on success. 1..7 are vpip::ErrorCode in declaration order
 *    (proj/include/vpip/error.hpp:23-31): 1 TooFewVertices, 2 NotConvex,
 *    3 DegenerateEdge, 4 NonFinite, 5 GeneratorCollision, 6 InvalidParameter,
 *    7 ParseError. 100 when the device is not an sm_100 part, 101 when
 *    libnccl.so.2 cannot be loaded, 200 + ncclResult_t for NCCL failures,
 *    1000 + cudaError_t for CUDA failures. No exception crosses the ABI.
 *  - `stream` is a cudaStream_t passed as void* (NULL = legacy default).
 *    Device-pointer calls are asynchronous on that stream; the caller owns
 *    point, mask and count buffers; the library owns a handle's tables.
 *  - Handles are immutable after prepare: any number of threads and streams
 *    may use one handle concurrently (engines.hpp:80-84).
 *  - Masks: `mask_words` holds ceil(m/32) little-endian u32 words; bit b of
 *    word w is point 32w+b. As a byte stream this is exactly the PIPM payload
 *    (io.cpp:272-279: bit j of the payload is point j, LSB-first).
 *    `mask_bytes` is the reference InclusionMask layout (engines.hpp:53-54):
 *    one byte per point, 1 = inside. Either may be NULL.
 *  - `d_inside` (device u64, may be NULL) is ACCUMULATED into: the fused
 *    count_inside (engines.cpp:215-217). Zero it before the first call.
 *  - dtype VPIPG_F64: the reference's own fp64 arithmetic, operation for
 *    operation (no FMA contraction) -> masks bit-identical to the reference.
 *    dtype VPIPG_F32: float32 points, fast affine kernels; masks equal the
 *    reference's on the same (f32-rounded) points for every point farther than
 *    1e-5 * max(1,|x|,|y|,extent) from every edge line.
 */
#ifndef VPIPG_H
#define VPIPG_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define VPIPG_ABI_VERSION 2

/* engines: vpip::EngineKind order (engines.hpp:64-73) */
#define VPIPG_ENGINE_VORONOI 0
#define VPIPG_ENGINE_OFFSET 1
#define VPIPG_ENGINE_CROSSING 2

/* preparation kinds (bit set) */
#define VPIPG_KIND_VORONOI (1u << 0)
#define VPIPG_KIND_OFFSET (1u << 1)
#define VPIPG_KIND_CROSSING (1u << 2)
#define VPIPG_KIND_ALL 7u

/* point dtypes */
#define VPIPG_F64 0
#define VPIPG_F32 1

#define VPIPG_ERR_ARCH 100
#define VPIPG_ERR_NCCL_MISSING 101
#define VPIPG_ERR_NCCL 200
#define VPIPG_ERR_CUDA 1000

typedef struct vpipg_poly vpipg_poly;

/* Human-readable text for a return code (error.hpp:33-45 for 1..7). */
const char* vpipg_strerror(int code);
int vpipg_abi_version(void);

/* Replaces: validate_polygon (geometry.cpp:53-98, geometry.hpp:110-111) +
 * to_voronoi (voronoi.cpp:60-71, voronoi.hpp:67-70) + the sign-of-offset and
 * ray-crossing per-edge setup hoisted out of engines.cpp:146-149, :176-186.
 * Vertices are host f64 arrays. When `kinds` includes VORONOI or OFFSET the
 * polygon is validated with the reference rules (error codes 1-4) and, for
 * VORONOI, converted on the device (centroid + one reflection per edge, the
 * reference's operation order; code 5 on a collision). CROSSING alone takes
 * the raw vertices unvalidated, any orientation (vpip.cpp:120-128).
 * Validation (codes 1-4) runs on the host before the call returns; the device
 * conversion is only ENQUEUED on `stream` (no synchronisation): its status
 * (code 5 on a collision) is returned by the first call that uses the handle,
 * or by vpipg_poly_status. */
int vpipg_prepare(const double* vx, const double* vy, uint32_t n, uint32_t kinds, int device,
                  void* stream, vpipg_poly** out);

/* Replaces the GeneratorSet argument of voronoi_contains_batch
 * (engines.hpp:90-96): a handle built from an explicit generator set
 * (inner point, n outer points) instead of a polygon. VORONOI only. */
int vpipg_prepare_generators(const double* inner_xy, const double* outer_xy, uint32_t n,
                             int device, void* stream, vpipg_poly** out);

/* Returns the handle's tables to the library's device pool (stream-ordered on
 * the legacy default stream, no device-wide synchronisation). Work that still
 * uses the handle on other streams must have completed. */
void vpipg_destroy(vpipg_poly* poly);

/* Waits for the handle's device conversion; 0 or its error code (5). */
int vpipg_poly_status(const vpipg_poly* poly);

/* n, prepared kinds, and whether validation reversed a clockwise input
 * (ConvexPolygon::was_reversed, geometry.hpp:95). Any pointer may be NULL. */
int vpipg_poly_info(const vpipg_poly* poly, uint32_t* n, uint32_t* kinds, int* reversed);

/* Reads back the generator set built on the device (GeneratorSet,
 * voronoi.hpp:58-65): inner_xy[2], outer_xy[2n]. Synchronous. */
int vpipg_poly_generators(const vpipg_poly* poly, double* inner_xy, double* outer_xy);

/* Reads back the validated CCW vertices (ConvexPolygon::vertices). */
int vpipg_poly_vertices(const vpipg_poly* poly, double* vx, double* vy);

/* Replaces voronoi_contains_batch (engines.cpp:243-254),
 * sign_of_offset_contains_batch (:320-329), ray_crossing_contains_batch
 * (:369-378) and count_inside (:215-217), fused. xs, ys, mask_words,
 * mask_bytes, d_inside are DEVICE pointers. Asynchronous on `stream`. */
int vpipg_test(const vpipg_poly* poly, int engine, int dtype, const void* xs, const void* ys,
               uint64_t m, uint32_t* mask_words, uint8_t* mask_bytes,
               unsigned long long* d_inside, void* stream);

/* Several engines over one device batch: mask_words / mask_bytes / d_inside
 * indexed by engine (arrays of 3, entries may be NULL). With all three engines
 * (float64 points, or float32 within the plan vpipg_test_multi_fused reports)
 * this is ONE fused kernel that reads every point once and tests it under
 * Voronoi, sign-of-offset and crossing in turn; otherwise the engines run one
 * after another. The masks and counts equal three vpipg_test calls either way
 * (bit-identical to the reference for float64). */
int vpipg_test_multi(const vpipg_poly* poly, uint32_t engines, int dtype, const void* xs,
                     const void* ys, uint64_t m, uint32_t* const* mask_words,
                     uint8_t* const* mask_bytes, unsigned long long* const* d_inside,
                     void* stream);

/* Nonzero when vpipg_test_multi would run this batch as ONE fused launch: all
 * three engines and either float64 points (the exact kernels, any n) or
 * float32 points in 16-byte-aligned buffers of at least one slice per warp
 * with a polygon of at most VPIPG_FUSE_MAX_N (96) edges whose tables fit the
 * kernel parameter bank or shared memory (above that the per-engine kernels
 * are faster); else 0. The value names the kernel: 2 for the small-polygon
 * kernel (float32, at most 12 vertices, single-section slab tables of one
 * form, word outputs only), 1 for the general fused kernels -- the route
 * depends on the outputs too, so the answer assumes 16-byte-aligned word
 * outputs and no byte outputs. Pure query: no device work. */
int vpipg_test_multi_fused(const vpipg_poly* poly, uint32_t engines, int dtype, const void* xs,
                           const void* ys, uint64_t m);

/* Same with HOST buffers (pageable or pinned): chunked host->device copies,
 * the test kernel and device->host mask copies are pipelined over three
 * streams on `device`, through a per-device staging area kept between
 * calls. Synchronous; *inside receives the count (may be NULL).
 * This is the path the vpip:: C++ shim uses. */
int vpipg_test_host(const vpipg_poly* poly, int engine, int dtype, const void* xs,
                    const void* ys, uint64_t m, uint32_t* mask_words, uint8_t* mask_bytes,
                    uint64_t* inside);

/* Several engines over one host batch: the points cross PCIe once per chunk
 * and each engine in the bit set `engines` (1 << VPIPG_ENGINE_*) tests them.
 * mask_words / mask_bytes / inside are indexed by engine (arrays of 3; any
 * entry, or the array itself, may be NULL). */
int vpipg_test_host_multi(const vpipg_poly* poly, uint32_t engines, int dtype, const void* xs,
                          const void* ys, uint64_t m, uint32_t* const* mask_words,
                          uint8_t* const* mask_bytes, uint64_t* inside);

/* Frees the per-device staging (chunk buffers and streams) the host-buffer
 * calls keep between calls; the next host call re-creates it. */
int vpipg_release_staging(int device);

/* Instrumented work counters of voronoi_contains_batch(..., BatchStats&)
 * (engines.cpp:256-273): the branch-free kernels perform exactly
 * (n+1)*m distance evaluations and n*m comparisons. */
int vpipg_voronoi_work(const vpipg_poly* poly, uint64_t m, uint64_t* distance_evaluations,
                       uint64_t* comparisons);

/* ---- engine cross-validation on the device (run_validation, bench.cpp:279-308) ---- */
#define VPIPG_REPORT_SAMPLES 100
typedef struct {
  uint64_t point_count;
  /* {voronoi/offset, voronoi/crossing, offset/crossing} (bench.hpp:91-92); for
   * vpipg_compare_masks: {a/b, a/b, 0} */
  uint64_t pair_disagreements[3];
  uint64_t disagreeing_points;
  /* disagreeing points farther than the band from every edge supporting line */
  uint64_t outside_band;
  int pass; /* outside_band == 0 */
  uint32_t n_samples;                           /* first disagreements by index */
  uint64_t sample_index[VPIPG_REPORT_SAMPLES];
  double sample_dist[VPIPG_REPORT_SAMPLES];     /* edge_line_distance (voronoi.cpp:73-82) */
  uint32_t sample_engines[VPIPG_REPORT_SAMPLES];/* bit0 voronoi, bit1 offset, bit2 crossing, bit3 outside band */
} vpipg_report;

/* All three engines on one batch (device pointers, f32 or f64), then every
 * disagreeing point's distance to the nearest edge line against `band`
 * (absolute, like tol::kAgreementBand, or relative: band * max(1, |x|, |y|,
 * polygon extent) when band_relative != 0). Needs a handle prepared with all
 * three kinds. Synchronous on `stream`. */
int vpipg_validate(const vpipg_poly* poly, int dtype, const void* xs, const void* ys, uint64_t m,
                   double band, int band_relative, vpipg_report* out, void* stream);

/* The same classification for two existing masks (device word arrays) of one
 * batch, e.g. the reference-exact f64 engine against the fp32 engine. */
int vpipg_compare_masks(const vpipg_poly* poly, int dtype, const void* xs, const void* ys,
                        uint64_t m, const uint32_t* words_a, const uint32_t* words_b, double band,
                        int band_relative, vpipg_report* out, void* stream);

/* ---- polygon database join (BASELINE config 4) ----
 * A CSR batch of polygons: polygon i owns vertices offsets[i] .. offsets[i+1]-1
 * of vx / vy (host arrays, f64). Replaces a loop of validate_polygon +
 * to_voronoi (geometry.cpp:53-98, voronoi.cpp:60-71) over the polygons with
 * one device kernel (one thread per polygon, the reference's exact f64
 * arithmetic). When `kinds` includes VORONOI or OFFSET every polygon is
 * validated; per_poly_status (host, npoly entries, may be NULL) receives 0 or
 * its vpip::ErrorCode + 1, and pairs that reference a failed polygon test
 * outside. Returns 0 when the table was built, even if some polygons failed. */
typedef struct vpipg_db vpipg_db;
int vpipg_prepare_csr(const uint32_t* offsets, const double* vx, const double* vy,
                      uint32_t npoly, uint32_t kinds, int device, void* stream, vpipg_db** out,
                      int32_t* per_poly_status);
void vpipg_db_destroy(vpipg_db* db);
int vpipg_db_info(const vpipg_db* db, uint32_t* npoly, uint64_t* nverts, uint32_t* kinds);
/* Generator set of polygon `poly` as built on the device (inner_xy[2], outer_xy[2n]). */
int vpipg_db_generators(const vpipg_db* db, uint32_t poly, double* inner_xy, double* outer_xy);

/* Gathered test: pair j tests point (xs[j], ys[j]) against polygon ids[j]
 * (float32 points, device pointers, asynchronous). Ids >= npoly test outside.
 * Same mask / count conventions as vpipg_test. */
int vpipg_test_gather(const vpipg_db* db, int engine, const float* xs, const float* ys,
                      const uint32_t* ids, uint64_t m, uint32_t* mask_words, uint8_t* mask_bytes,
                      unsigned long long* d_inside, void* stream);

/* All requested engines over one batch of (point, polygon id) pairs:
 * mask_words / mask_bytes / d_inside indexed by engine (arrays of 3, entries
 * may be NULL). With all three engines this is ONE fused kernel that reads
 * every pair once and walks two polygon blocks per pair instead of three
 * (sign-of-offset and crossing share the vertex rows); results equal three
 * vpipg_test_gather calls. Asynchronous on `stream`. */
int vpipg_test_gather_multi(const vpipg_db* db, uint32_t engines, const float* xs, const float* ys,
                            const uint32_t* ids, uint64_t m, uint32_t* const* mask_words,
                            uint8_t* const* mask_bytes, unsigned long long* const* d_inside,
                            void* stream);

/* The join over HOST buffers (pageable or pinned): every engine in the bit set
 * `engines` over one copy of the pairs, chunked and pipelined like
 * vpipg_test_host_multi (mask_words / mask_bytes / inside indexed by engine,
 * arrays of 3, entries may be NULL). Synchronous. */
int vpipg_test_gather_host(const vpipg_db* db, uint32_t engines, const float* xs, const float* ys,
                           const uint32_t* ids, uint64_t m, uint32_t* const* mask_words,
                           uint8_t* const* mask_bytes, uint64_t* inside);

/* Join-pair workload generator (input generation, not timed): pair j gets
 * id = floor(U(seed, 3j) * npoly) and point = centre[id] + (2U - 1) * radius[id]
 * per axis (U from mix_seed(seed, 3j+1 / 3j+2)), rounded to f32. centre_x,
 * centre_y, radius: device f64 arrays of npoly entries. */
int vpipg_fill_join_pairs(uint64_t seed, uint64_t first, uint64_t m, uint32_t npoly,
                          const double* centre_x, const double* centre_y, const double* radius,
                          float* xs, float* ys, uint32_t* ids, void* stream);

/* Counter-based uniform points on the device: point j (j = first..first+m-1)
 * is (min_x + w*U(mix_seed(seed, 2j)), min_y + h*U(mix_seed(seed, 2j+1))),
 * U = top-53-bit uniform (sampling.cpp:31-33), mix_seed = sampling.cpp:107-112,
 * stored as f64 or rounded to f32. Input generation, not timed work. */
int vpipg_fill_uniform_points(uint64_t seed, uint64_t first, uint64_t m, double min_x,
                              double min_y, double max_x, double max_y, int dtype, void* xs,
                              void* ys, void* stream);

/* ---- Multi-GPU: the inside-count all-reduce -------------
 * Points shard across GPUs with no data exchange; the one collective of the
 * path is a sum of the per-GPU inside counts (3 u64 for the three engines),
 * launched on the test kernels' stream right after them (graph-capturable).
 * NCCL is loaded at run time (dlopen "libnccl.so.2", or $VPIPG_NCCL_LIBRARY),
 * so the library itself has no link-time NCCL dependency.
 *
 * One process per GPU: rank 0 calls vpipg_comm_unique_id, ships the 128 bytes
 * to the other ranks out of band (torch.distributed, MPI, a file), and every
 * rank calls vpipg_comm_init. One process driving several GPUs:
 * vpipg_comm_init_all, then vpipg_allreduce_counts_group from one thread. */
typedef struct vpipg_comm vpipg_comm;

/* NCCL_VERSION_CODE of the loaded libnccl (e.g. 22809 for 2.28.9). */
int vpipg_nccl_version(int* version);
int vpipg_comm_unique_id(uint8_t id[128]);
int vpipg_comm_init(const uint8_t id[128], int nranks, int rank, int device, vpipg_comm** out);
int vpipg_comm_init_all(int ndev, const int* devices, vpipg_comm** comms);
int vpipg_comm_info(const vpipg_comm* comm, int* nranks, int* rank, int* device);
/* Zero n device u64 counters on `stream` (a memset, no kernel launch; the
 * test calls accumulate into their d_inside counters). */
int vpipg_zero_counts(unsigned long long* d_counts, int n, void* stream);
/* In-place sum of n device u64 counters over all ranks, on `stream`. */
int vpipg_allreduce_counts(vpipg_comm* comm, unsigned long long* d_counts, int n, void* stream);
/* The same for several communicators driven by one thread (vpipg_comm_init_all):
 * comms[i], d_counts[i], streams[i] belong to the same device. */
int vpipg_allreduce_counts_group(int ncomms, vpipg_comm* const* comms,
                                 unsigned long long* const* d_counts, int n,
                                 void* const* streams);
int vpipg_comm_destroy(vpipg_comm* comm);

/* Host-side seeded polygon and point samplers with the reference's exact
 * semantics (sampling.cpp:50-105), for building workloads. Vertices come
 * back validated (CCW). */
uint64_t vpipg_mix_seed(uint64_t seed, uint64_t salt);
int vpipg_regular_polygon(uint32_t n, double r, double cx, double cy, double* vx, double* vy);
int vpipg_random_convex_polygon(uint32_t n, uint64_t seed, double r, double cx, double cy,
                                double* vx, double* vy);
int vpipg_sample_points(uint64_t count, double min_x, double min_y, double max_x, double max_y,
                        uint64_t seed, double* xs, double* ys);

#ifdef __cplusplus
}
#endif
#endif /* VPIPG_H */
