// vpipg_internal.h -- host/device shared declarations inside libvpipg.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "vpipg_device.cuh"

namespace vpipg {

constexpr uint32_t kKindVoronoi = 1u;
constexpr uint32_t kKindOffset = 2u;
constexpr uint32_t kKindCrossing = 4u;

struct PrepArgs {
  const double* vv;      // validated CCW vertices [x0..x(n-1), y0..y(n-1)] or null
  const double* vr;      // raw vertices (crossing) in the same layout, or null
  const double* gen_in;  // explicit generator set [ix, iy, ox0, oy0, ...] or null
  uint32_t n;
  uint32_t kinds;
  double2* outer;
  OffsetEdgeF64* off;
  RayEdgeF64* ray;
  float2* slab_coef[2];  // capacity n + 4 entries each
  float4* cross_vert;
  double4* lines;        // n unit-normal edge lines (band metric)
  PrepMeta* meta;
  // the handle's pinned, mapped host block: the kernel copies the final
  // PrepMeta there and, when tables_out, the slab tables (n + 4 pairs each)
  // and the crossing table at the given byte offsets (no download call)
  char* host_out;
  uint32_t out_slab[2], out_cross;
  int tables_out;
};

// Small prepare inputs in the prep kernel's parameter bank (no upload call):
// vv / vr / gen laid out in v[], offsets in doubles, -1 = absent.
constexpr int kPrepInlineMax = 512;
struct PrepInline {
  int32_t vv_at = -1, vr_at = -1, gen_at = -1, pad_ = 0;
  double v[kPrepInlineMax];
};

struct TestArgs {
  const void* xs;
  const void* ys;
  uint64_t m;
  uint32_t* words;
  uint8_t* bytes;
  unsigned long long* inside;
};

// ---- polygon database (CSR batch of polygons; csr.cu) ----
constexpr uint32_t kRangeInvalid = 0x80000000u;  // polygon failed validation: Voronoi / offset outside
constexpr uint32_t kReversed = 0x40000000u;      // validation reversed the (clockwise) raw order
constexpr uint32_t kNMask = 0x3fffffffu;

// ONE record per polygon, 32-byte aligned, at float2 slot 4 * rec[i] (rec[i] =
// i * stride when the database uses a fixed stride):
//   slot 0   (n | kRangeInvalid | kReversed as u32 bits, 0)
//   slot 1   frame origin c (f32 centre of the bounding box)
//   slot 2   p0' = centroid - c (f32; the Voronoi inner generator)
//   slot 3   v_{n-1}' (closes the ring)
//   slot 4 + k  the row v_k' (f32, relative to c) in the VALIDATED
//            (counter-clockwise) order, padded with copies of v_{n-1}' to
//            whole 4-row (32-byte) chunks, at least two chunks per record
// so a pair reads one header and one walk of n rows for all three engines:
// sign-of-offset and Voronoi in the validated order the reference tests them
// in, the crossing on the same rows (for a clockwise raw polygon that is the
// raw ring travelled backwards, which leaves the crossing parity unchanged),
// Voronoi with each outer generator rebuilt in registers from its edge's two
// rows and p0' (12.125 bytes of stream and ~4.3 32-byte sectors of record per
// C4 pair).
struct CsrPrepArgs {
  const uint32_t* offsets;  // npoly + 1 (input CSR)
  const double* vx;         // raw vertices (device)
  const double* vy;
  uint32_t npoly;
  uint32_t kinds;
  const uint32_t* rec;      // npoly record offsets, 32-byte units
  double2* inner;           // npoly generators (f64, exact)
  double2* outer;           // nverts generators (f64, exact), input CSR layout (validated order)
  float2* recs;             // the records
  int32_t* status;          // npoly: 0 or ErrorCode + 1
};

struct DbTables {
  uint32_t npoly;
  uint32_t kinds;
  uint32_t stride;        // > 0: record i at 32-byte unit i * stride; 0: at rec[i]
  const uint32_t* rec;
  const float2* recs;
};

struct GatherArgs {
  const float* xs;
  const float* ys;
  const uint32_t* ids;
  uint64_t m;
  uint32_t* words;
  uint8_t* bytes;
  unsigned long long* inside;
};

cudaError_t launch_prep(const PrepArgs& args, const PrepInline* in, cudaStream_t stream);
cudaError_t launch_prep_csr(const CsrPrepArgs& args, cudaStream_t stream);
cudaError_t launch_gather(const DbTables& t, int engine, const GatherArgs& a, cudaStream_t stream);
// all three engines per pair in one pass (a[0..2] share xs, ys, ids, m)
cudaError_t launch_gather_all(const DbTables& t, const GatherArgs* a, cudaStream_t stream);
cudaError_t launch_fill_pairs(uint64_t seed, uint64_t first, uint64_t m, uint32_t npoly,
                              const double* cx, const double* cy, const double* rad, float* xs,
                              float* ys, uint32_t* ids, cudaStream_t stream);
cudaError_t launch_test_f32(const DevTables& t, int engine, const TestArgs& a, cudaStream_t stream);
// all three engines in one fused pass over the points (a[0..2] share xs, ys,
// m); cudaErrorNotSupported when the tables or the batch do not fit its plan
cudaError_t launch_test_f32_all(const DevTables& t, const TestArgs* a, cudaStream_t stream);
// fp64: all three engines in one pass (reference-exact, any n)
cudaError_t launch_test_f64_all(const DevTables& t, const TestArgs* a, cudaStream_t stream);
// whether launch_test_f32_all takes this batch as one fused launch
bool test_f32_all_plan(const DevTables& t, const TestArgs* a, size_t* smem);
// the small-polygon fused kernel (tri_small.cu): at most 8 crossing vertices,
// single-section slab tables of one form, 16-byte aligned points and word
// outputs, no byte outputs; cudaErrorNotSupported otherwise
bool test_f32_small_plan(const DevTables& t, const TestArgs* a);
cudaError_t launch_test_f32_small(const DevTables& t, const TestArgs* a, cudaStream_t stream);
cudaError_t launch_test_f64(const DevTables& t, int engine, const TestArgs& a, cudaStream_t stream);
// ---- validation (validate.cu): run_validation (bench.cpp:279-308) on the device ----
constexpr int kReportSamples = 100;
constexpr uint32_t kSampleCapacity = 1u << 16;
struct ReportDev {                    // device-side accumulators
  unsigned long long pair[3];         // voronoi/offset, voronoi/crossing, offset/crossing
  unsigned long long disagreeing;
  unsigned long long outside_band;
  unsigned long long n_recorded;
  unsigned long long sample_index[kSampleCapacity];
  double sample_dist[kSampleCapacity];
  uint32_t sample_bits[kSampleCapacity];  // engine mask bits v | s << 1 | c << 2
};
struct ClassifyArgs {
  const uint32_t* w[3];  // mask words per engine (w[2] may be null: two-mask compare)
  const void* xs;
  const void* ys;
  int dtype;
  uint64_t m;
  double band;
  int relative;          // band * max(1, |x|, |y|, extent) when set
  double extent;
  const double4* lines;
  uint32_t n;
  ReportDev* rep;
};
cudaError_t launch_classify(const ClassifyArgs& a, cudaStream_t stream);
cudaError_t launch_fill_uniform(uint64_t seed, uint64_t first, uint64_t m, double min_x,
                                double min_y, double max_x, double max_y, int dtype, void* xs,
                                void* ys, cudaStream_t stream);

// Launch configuration cache (capi.cu): for `kernel` on the current device,
// raises its dynamic shared-memory limit to `smem` if no earlier launch did,
// and returns the SM count and resident blocks per SM for (threads, smem) --
// the driver queries run once per (device, kernel, threads, smem).
cudaError_t launch_config(const void* kernel, int threads, size_t smem, int* sms, int* per_sm);

}  // namespace vpipg

// comm.cpp: text for a VPIPG_ERR_NCCL + ncclResult_t code
const char* vpipg_nccl_error_string(int code);
