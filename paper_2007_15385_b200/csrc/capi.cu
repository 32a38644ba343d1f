// capi.cu -- host side of the C-ABI (include/vpipg.h).
//
// Owns handle lifetime, host-side polygon validation (the reference's
// precondition, geometry.cpp:53-98, restated exactly), blob layout, kernel
// dispatch, the polygon database and device-side validation; the host-buffer
// calls live in hostpipe.cu. No compute on the point
// stream happens here: every point test runs in a device kernel, and a
// missing or wrong-architecture device is an error (no CPU fallback).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <new>
#include <numbers>
#include <random>
#include <tuple>
#include <vector>

#include "capi_internal.h"
#include "exact_geom.cuh"

using namespace vpipg;
using namespace vpipg::capi;

namespace {

// The kernels are built for sm_100a only; refuse anything else loudly.
int check_device(int device) {
  static std::mutex mu;
  static std::vector<int> ok(64, -1);
  if (device < 0 || device >= 64) return kInvalid;
  std::lock_guard<std::mutex> lock(mu);
  if (ok[device] < 0) {
    cudaDeviceProp prop;
    const cudaError_t e = cudaGetDeviceProperties(&prop, device);
    if (e != cudaSuccess) return cuda_code(e);
    ok[device] = (prop.major == 10 && prop.minor == 0) ? 1 : 0;
  }
  return ok[device] ? kOk : VPIPG_ERR_ARCH;
}

// validate_polygon (geometry.cpp:53-98) on the host: exact_geom.cuh's
// validate_exact, the same definition the device CSR ingest runs; reverses the
// vertices in place when they are clockwise.
int validate(std::vector<double>& vx, std::vector<double>& vy, int* reversed) {
  bool rev = false;
  const int rc = validate_exact([&](int k) { return make_double2(vx[k], vy[k]); },
                                static_cast<int>(vx.size()), &rev);
  *reversed = rev ? 1 : 0;
  if (rc == 0 && rev) {
    std::reverse(vx.begin(), vx.end());
    std::reverse(vy.begin(), vy.end());
  }
  return rc;
}


// Per-device pool for polygon blobs: memory stays cached in the pool between
// prepares (release threshold = max), so prepare / destroy cost no cudaMalloc /
// cudaFree and no device-wide synchronisation.
int blob_pool(int device, cudaMemPool_t* out) {
  static std::mutex mu;
  static cudaMemPool_t pools[64] = {};
  std::lock_guard<std::mutex> lock(mu);
  if (!pools[device]) {
    cudaMemPoolProps props{};
    props.allocType = cudaMemAllocationTypePinned;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = device;
    VPIPG_TRY(cudaMemPoolCreate(&pools[device], &props));
    uint64_t keep = UINT64_MAX;
    VPIPG_TRY(cudaMemPoolSetAttribute(pools[device], cudaMemPoolAttrReleaseThreshold, &keep));
  }
  *out = pools[device];
  return kOk;
}

constexpr uint32_t kHostTableMax = 256;

// Pinned host blocks for the asynchronous prepare (uploads and the download of
// the status and f32 tables): power-of-two size classes carved from 4 MiB
// cudaHostAlloc chunks and recycled, so a prepare makes no pinned allocation
// once warm. Portable across devices.
class PinnedArena {
 public:
  static PinnedArena& get() {
    static PinnedArena a;
    return a;
  }
  char* take(size_t bytes, size_t* got) {
    int cls = 12;  // 4 KiB minimum
    while ((size_t(1) << cls) < bytes) ++cls;
    const size_t size = size_t(1) << cls;
    std::lock_guard<std::mutex> lock(mu_);
    auto& fl = free_[cls];
    if (!fl.empty()) {
      char* b = fl.back();
      fl.pop_back();
      *got = size;
      return b;
    }
    if (size > kChunk) {  // large: its own allocation
      void* h = nullptr;
      if (cudaHostAlloc(&h, size, cudaHostAllocPortable | cudaHostAllocMapped) != cudaSuccess)
        return nullptr;
      *got = size;
      return static_cast<char*>(h);
    }
    if (left_ < size) {
      void* h = nullptr;
      if (cudaHostAlloc(&h, kChunk, cudaHostAllocPortable | cudaHostAllocMapped) != cudaSuccess)
        return nullptr;
      cur_ = static_cast<char*>(h);
      left_ = kChunk;
    }
    char* b = cur_;
    cur_ += size;
    left_ -= size;
    *got = size;
    return b;
  }
  void give(char* b, size_t size) {
    if (!b) return;
    int cls = 12;
    while ((size_t(1) << cls) < size) ++cls;
    std::lock_guard<std::mutex> lock(mu_);
    free_[cls].push_back(b);
  }

 private:
  static constexpr size_t kChunk = size_t(4) << 20;
  std::mutex mu_;
  std::map<int, std::vector<char*>> free_;
  char* cur_ = nullptr;
  size_t left_ = 0;
};

// Per-device pool of cudaEventDisableTiming events for the prepare handles.
class EventPool {
 public:
  static EventPool& get() {
    static EventPool p;
    return p;
  }
  cudaEvent_t take(int device) {
    {
      std::lock_guard<std::mutex> lock(mu_);
      auto& v = free_[device];
      if (!v.empty()) {
        cudaEvent_t e = v.back();
        v.pop_back();
        return e;
      }
    }
    cudaEvent_t e = nullptr;
    return cudaEventCreateWithFlags(&e, cudaEventDisableTiming) == cudaSuccess ? e : nullptr;
  }
  void give(int device, cudaEvent_t e) {
    if (!e) return;
    std::lock_guard<std::mutex> lock(mu_);
    free_[device].push_back(e);
  }

 private:
  std::mutex mu_;
  std::map<int, std::vector<cudaEvent_t>> free_;
};

// Builds the blob and enqueues the prep kernel: uploads from a pinned block,
// downloads the status, slab counts and (small) f32 tables into it, records
// the handle's event. Nothing waits here; ensure_ready finishes the handle.
int build(vpipg_poly* p, const double* vv, const double* vr, const double* gen, cudaStream_t s) {
  const size_t n = p->n;
  size_t off = 0;
  auto take = [&](size_t bytes) { const size_t o = off; off = align256(off + bytes); return o; };
  const size_t o_vv = take(2 * n * sizeof(double));
  const size_t o_vr = take(2 * n * sizeof(double));
  const size_t o_gen = take((2 + 2 * n) * sizeof(double));
  const size_t o_outer = take(n * sizeof(double2));
  const size_t o_off = take(n * sizeof(OffsetEdgeF64));
  const size_t o_ray = take(n * sizeof(RayEdgeF64));
  const size_t o_lines = take(n * sizeof(double4));
  // the download span: status + counts, then the f32 tables, contiguous
  const size_t o_meta = take(sizeof(PrepMeta));
  const size_t o_s0 = take((n + 4) * sizeof(float2));
  const size_t o_s1 = take((n + 4) * sizeof(float2));
  const size_t o_cross = take(n * sizeof(float4));
  const size_t o_end = off;
  p->host_tables = n <= kHostTableMax;
  const size_t dl = p->host_tables ? o_end - o_meta : o_s0 - o_meta;
  p->host = PinnedArena::get().take(o_outer + dl, &p->host_bytes);
  if (!p->host) return kInvalid;
  p->dl_meta = o_outer;
  p->dl_slab[0] = o_outer + (o_s0 - o_meta);
  p->dl_slab[1] = o_outer + (o_s1 - o_meta);
  p->dl_cross = o_outer + (o_cross - o_meta);
  p->ready = EventPool::get().take(p->device);
  if (!p->ready) return kInvalid;
  // stream-ordered allocation from the library's per-device pool (no device
  // synchronisation on prepare / destroy), one packed upload of the inputs
  cudaMemPool_t pool = nullptr;
  int rc = blob_pool(p->device, &pool);
  if (rc) return rc;
  VPIPG_TRY(cudaMallocFromPoolAsync(&p->blob, off, pool, s));
  char* b = static_cast<char*>(p->blob);
  PrepArgs& a = p->args;
  a.n = p->n;
  a.kinds = p->kinds;
  // small inputs ride in the prep kernel's parameters; larger ones are one
  // upload from the pinned block in the blob's own layout [vv | vr | gen]
  const size_t need = (vv ? 2 * n : 0) + (vr ? 2 * n : 0) + (gen ? 2 + 2 * n : 0);
  PrepInline inl;
  const bool inline_in = need <= size_t(kPrepInlineMax);
  if (inline_in) {
    int32_t at = 0;
    auto put = [&](const double* src, size_t cnt, int32_t* where) {
      if (!src) return;
      std::memcpy(inl.v + at, src, cnt * sizeof(double));
      *where = at;
      at += static_cast<int32_t>(cnt);
    };
    put(vv, 2 * n, &inl.vv_at);
    put(vr, 2 * n, &inl.vr_at);
    put(gen, 2 + 2 * n, &inl.gen_at);
  } else {
    char* up = p->host;
    if (vv) {
      std::memcpy(up + o_vv, vv, 2 * n * sizeof(double));
      a.vv = reinterpret_cast<const double*>(b + o_vv);
    }
    if (vr) {
      std::memcpy(up + o_vr, vr, 2 * n * sizeof(double));
      a.vr = reinterpret_cast<const double*>(b + o_vr);
    }
    if (gen) {
      std::memcpy(up + o_gen, gen, (2 + 2 * n) * sizeof(double));
      a.gen_in = reinterpret_cast<const double*>(b + o_gen);
    }
    if (o_outer) VPIPG_TRY(cudaMemcpyAsync(b, up, o_outer, cudaMemcpyHostToDevice, s));
  }
  a.outer = reinterpret_cast<double2*>(b + o_outer);
  a.off = reinterpret_cast<OffsetEdgeF64*>(b + o_off);
  a.ray = reinterpret_cast<RayEdgeF64*>(b + o_ray);
  a.slab_coef[0] = reinterpret_cast<float2*>(b + o_s0);
  a.slab_coef[1] = reinterpret_cast<float2*>(b + o_s1);
  a.cross_vert = reinterpret_cast<float4*>(b + o_cross);
  a.lines = reinterpret_cast<double4*>(b + o_lines);
  a.meta = reinterpret_cast<PrepMeta*>(b + o_meta);
  // the kernel writes the status, counts and small tables straight into the
  // mapped pinned block (unified addressing: the host pointer is valid on the
  // device), so no download call is enqueued
  (void)dl;
  a.host_out = p->host + p->dl_meta;
  a.out_slab[0] = static_cast<uint32_t>(o_s0 - o_meta);
  a.out_slab[1] = static_cast<uint32_t>(o_s1 - o_meta);
  a.out_cross = static_cast<uint32_t>(o_cross - o_meta);
  a.tables_out = p->host_tables ? 1 : 0;
  VPIPG_TRY(launch_prep(a, inline_in ? &inl : nullptr, s));
  VPIPG_TRY(cudaEventRecord(p->ready, s));
  p->state.store(-1, std::memory_order_release);
  return kOk;
}

}  // namespace

int vpipg::capi::ensure_ready(const vpipg_poly* p) {
  int st = p->state.load(std::memory_order_acquire);
  if (st >= 0) return st;
  std::lock_guard<std::mutex> lock(p->mu);
  st = p->state.load(std::memory_order_relaxed);
  if (st >= 0) return st;
  DeviceGuard g(p->device);
  const cudaError_t e = cudaEventSynchronize(p->ready);
  if (e != cudaSuccess) return cuda_code(e);  // stays pending: a later call retries
  PrepMeta meta;
  std::memcpy(&meta, p->host + p->dl_meta, sizeof(meta));
  if (meta.status != 0) {
    p->state.store(meta.status, std::memory_order_release);
    return meta.status;
  }
  const PrepArgs& a = p->args;
  DevTables& t = p->t;
  t.n = p->n;
  t.kinds = p->kinds;
  t.inner_x = meta.inner_x;
  t.inner_y = meta.inner_y;
  t.outer = a.outer;
  t.off = a.off;
  t.ray = a.ray;
  t.ox = meta.ox;
  t.oy = meta.oy;
  for (int k = 0; k < 2; ++k) {
    SlabTable& stb = t.slab[k];
    stb.coef = a.slab_coef[k];
    uint32_t acc = 0;
    for (int gi = 0; gi < kGroups; ++gi) {
      stb.off[gi] = acc;
      stb.cnt[gi] = meta.cnt[k][gi];
      acc += meta.cnt[k][gi];
    }
    stb.total = acc;
    // small tables also travel in the kernels' parameter bank (test_f32.cu)
    t.h_slab[k] = p->host_tables ? reinterpret_cast<const float2*>(p->host + p->dl_slab[k]) : nullptr;
  }
  t.cross.vert = a.cross_vert;
  t.cross.n = p->n;
  t.h_cross = p->host_tables ? reinterpret_cast<const float4*>(p->host + p->dl_cross) : nullptr;
  t.lines = a.lines;
  p->inner_x = meta.inner_x;
  p->inner_y = meta.inner_y;
  p->state.store(0, std::memory_order_release);
  return 0;
}

int vpipg::capi::dispatch(const vpipg_poly* p, int engine, int dtype, const TestArgs& a,
                          cudaStream_t s) {
  const uint32_t need = engine == VPIPG_ENGINE_VORONOI  ? kKindVoronoi
                        : engine == VPIPG_ENGINE_OFFSET ? kKindOffset
                        : engine == VPIPG_ENGINE_CROSSING ? kKindCrossing
                                                          : 0u;
  if (need == 0 || !(p->kinds & need)) return kInvalid;
  if (dtype != VPIPG_F32 && dtype != VPIPG_F64) return kInvalid;
  if (const int st = ensure_ready(p)) return st;
  if (a.m == 0) return kOk;
  if (!a.xs || !a.ys) return kInvalid;
  const cudaError_t e = (dtype == VPIPG_F32) ? launch_test_f32(p->t, engine, a, s)
                                             : launch_test_f64(p->t, engine, a, s);
  return cuda_code(e);
}


extern "C" {

const char* vpipg_strerror(int code) {
  switch (code) {
    case 0: return "ok";
    case 1: return "too few vertices";
    case 2: return "not convex";
    case 3: return "degenerate edge";
    case 4: return "non-finite value";
    case 5: return "generator collision";
    case 6: return "invalid parameter";
    case 7: return "parse error";
    case VPIPG_ERR_ARCH: return "device is not an sm_100 (B200) GPU";
    case VPIPG_ERR_NCCL_MISSING: return "libnccl.so.2 could not be loaded";
    default: break;
  }
  if (code > VPIPG_ERR_NCCL && code < VPIPG_ERR_NCCL + 100) return vpipg_nccl_error_string(code);
  if (code > VPIPG_ERR_CUDA)
    return cudaGetErrorString(static_cast<cudaError_t>(code - VPIPG_ERR_CUDA));
  return "unknown error";
}

int vpipg_abi_version(void) { return VPIPG_ABI_VERSION; }

int vpipg_prepare(const double* vx, const double* vy, uint32_t n, uint32_t kinds, int device,
                  void* stream, vpipg_poly** out) {
  if (!out || (kinds & ~VPIPG_KIND_ALL) || kinds == 0) return kInvalid;
  if (n > 0 && (!vx || !vy)) return kInvalid;
  *out = nullptr;
  int rc = check_device(device);
  if (rc) return rc;
  auto* p = new (std::nothrow) vpipg_poly;
  if (!p) return kInvalid;
  p->device = device;
  p->n = n;
  p->kinds = kinds;
  std::vector<double> raw(2 * size_t(n)), val;
  std::copy(vx, vx + n, raw.begin());
  std::copy(vy, vy + n, raw.begin() + n);
  const bool convex = kinds & (kKindVoronoi | kKindOffset);
  if (convex) {
    p->vx.assign(vx, vx + n);
    p->vy.assign(vy, vy + n);
    rc = validate(p->vx, p->vy, &p->reversed);
    if (rc) {
      delete p;
      return rc;
    }
    val.resize(2 * size_t(n));
    std::copy(p->vx.begin(), p->vx.end(), val.begin());
    std::copy(p->vy.begin(), p->vy.end(), val.begin() + n);
  } else {
    p->vx.assign(vx, vx + n);
    p->vy.assign(vy, vy + n);
  }
  DeviceGuard g(device);
  rc = build(p, convex ? val.data() : nullptr, (kinds & kKindCrossing) ? raw.data() : nullptr,
             nullptr, static_cast<cudaStream_t>(stream));
  if (rc) {
    vpipg_destroy(p);
    return rc;
  }
  *out = p;
  return kOk;
}

int vpipg_prepare_generators(const double* inner_xy, const double* outer_xy, uint32_t n,
                             int device, void* stream, vpipg_poly** out) {
  if (!out || !inner_xy || (n > 0 && !outer_xy)) return kInvalid;
  *out = nullptr;
  int rc = check_device(device);
  if (rc) return rc;
  auto* p = new (std::nothrow) vpipg_poly;
  if (!p) return kInvalid;
  p->device = device;
  p->n = n;
  p->kinds = kKindVoronoi;
  std::vector<double> gen(2 + 2 * size_t(n));
  gen[0] = inner_xy[0];
  gen[1] = inner_xy[1];
  std::copy(outer_xy, outer_xy + 2 * size_t(n), gen.begin() + 2);
  DeviceGuard g(device);
  rc = build(p, nullptr, nullptr, gen.data(), static_cast<cudaStream_t>(stream));
  if (rc) {
    vpipg_destroy(p);
    return rc;
  }
  *out = p;
  return kOk;
}

void vpipg_destroy(vpipg_poly* p) {
  if (!p) return;
  if (p->ready) {
    // the download into the pinned block may still be in flight
    DeviceGuard g(p->device);
    cudaEventSynchronize(p->ready);
    EventPool::get().give(p->device, p->ready);
  }
  PinnedArena::get().give(p->host, p->host_bytes);
  if (p->blob) {
    // back to the pool, ordered after all work on the legacy default stream;
    // work the caller still has in flight on other streams must be finished
    // (as with any buffer the caller frees)
    DeviceGuard g(p->device);
    cudaFreeAsync(p->blob, nullptr);
  }
  delete p;
}

int vpipg_poly_status(const vpipg_poly* p) {
  if (!p) return kInvalid;
  return ensure_ready(p);
}

int vpipg_poly_info(const vpipg_poly* p, uint32_t* n, uint32_t* kinds, int* reversed) {
  if (!p) return kInvalid;
  if (n) *n = p->n;
  if (kinds) *kinds = p->kinds;
  if (reversed) *reversed = p->reversed;
  return kOk;
}

int vpipg_poly_generators(const vpipg_poly* p, double* inner_xy, double* outer_xy) {
  if (!p || !(p->kinds & kKindVoronoi) || !inner_xy || (p->n && !outer_xy)) return kInvalid;
  DeviceGuard g(p->device);
  if (const int st = ensure_ready(p)) return st;
  inner_xy[0] = p->inner_x;
  inner_xy[1] = p->inner_y;
  if (p->n) VPIPG_TRY(cudaMemcpy(outer_xy, p->t.outer, p->n * sizeof(double2), cudaMemcpyDeviceToHost));
  return kOk;
}

int vpipg_poly_vertices(const vpipg_poly* p, double* vx, double* vy) {
  if (!p || (p->n && (!vx || !vy))) return kInvalid;
  std::copy(p->vx.begin(), p->vx.end(), vx);
  std::copy(p->vy.begin(), p->vy.end(), vy);
  return kOk;
}

int vpipg_test(const vpipg_poly* p, int engine, int dtype, const void* xs, const void* ys,
               uint64_t m, uint32_t* mask_words, uint8_t* mask_bytes,
               unsigned long long* d_inside, void* stream) {
  if (!p) return kInvalid;
  DeviceGuard g(p->device);
  TestArgs a{xs, ys, m, mask_words, mask_bytes, d_inside};
  return dispatch(p, engine, dtype, a, static_cast<cudaStream_t>(stream));
}

int vpipg_test_multi(const vpipg_poly* p, uint32_t engines, int dtype, const void* xs,
                     const void* ys, uint64_t m, uint32_t* const* mask_words,
                     uint8_t* const* mask_bytes, unsigned long long* const* d_inside,
                     void* stream) {
  if (!p || engines == 0 || (engines & ~7u)) return kInvalid;
  DeviceGuard g(p->device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  TestArgs a[3];
  for (int e = 0; e < 3; ++e)
    a[e] = TestArgs{xs, ys, m, mask_words ? mask_words[e] : nullptr,
                    mask_bytes ? mask_bytes[e] : nullptr, d_inside ? d_inside[e] : nullptr};
  if (engines == 7u && (p->kinds & VPIPG_KIND_ALL) == VPIPG_KIND_ALL && m > 0 && xs && ys) {
    if (const int st = ensure_ready(p)) return st;
    if (dtype == VPIPG_F64) return cuda_code(launch_test_f64_all(p->t, a, s));
    if (dtype == VPIPG_F32) {
      const cudaError_t e = launch_test_f32_all(p->t, a, s);
      if (e != cudaErrorNotSupported) return cuda_code(e);
    }
  }
  for (int e = 0; e < 3; ++e)  // one engine at a time
    if (engines & (1u << e)) {
      const int rc = dispatch(p, e, dtype, a[e], s);
      if (rc) return rc;
    }
  return kOk;
}

int vpipg_zero_counts(unsigned long long* d_counts, int n, void* stream) {
  if (n < 0 || (n > 0 && !d_counts)) return kInvalid;
  if (n == 0) return kOk;
  return cuda_code(cudaMemsetAsync(d_counts, 0, static_cast<size_t>(n) * sizeof(unsigned long long),
                                   static_cast<cudaStream_t>(stream)));
}

int vpipg_test_multi_fused(const vpipg_poly* p, uint32_t engines, int dtype, const void* xs,
                           const void* ys, uint64_t m) {
  if (!p || engines != 7u || (p->kinds & VPIPG_KIND_ALL) != VPIPG_KIND_ALL || m == 0 || !xs || !ys)
    return 0;
  if (dtype == VPIPG_F64) return 1;  // the exact kernels fuse at any n
  if (dtype != VPIPG_F32) return 0;
  TestArgs a[3];
  for (auto& x : a) x = TestArgs{xs, ys, m, nullptr, nullptr, nullptr};
  if (ensure_ready(p)) return 0;
  if (test_f32_small_plan(p->t, a)) return 2;
  return test_f32_all_plan(p->t, a, nullptr) ? 1 : 0;
}

int vpipg_prepare_csr(const uint32_t* offsets, const double* vx, const double* vy,
                      uint32_t npoly, uint32_t kinds, int device, void* stream, vpipg_db** out,
                      int32_t* per_poly_status) {
  if (!out || !offsets || (kinds & ~VPIPG_KIND_ALL) || kinds == 0) return kInvalid;
  *out = nullptr;
  if (offsets[0] != 0) return kInvalid;
  for (uint32_t i = 0; i < npoly; ++i)
    if (offsets[i + 1] < offsets[i]) return kInvalid;
  const uint64_t nv = offsets[npoly];
  if (nv && (!vx || !vy)) return kInvalid;
  int rc = check_device(device);
  if (rc) return rc;
  DeviceGuard g(device);
  auto* db = new (std::nothrow) vpipg_db;
  if (!db) return kInvalid;
  db->device = device;
  db->npoly = npoly;
  db->nverts = nv;
  db->kinds = kinds;
  db->offsets.assign(offsets, offsets + npoly + 1);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  // one 32-byte-aligned record per polygon, packed back to back: the header
  // (4 slots) and n rows, rounded up to whole 32-byte units (vpipg_internal.h)
  // (a fixed stride of the largest record when that costs at most 1.5x the
  // packed size -- C4's 4..16-gons -- saving the kernels a dependent load;
  // packed with per-polygon offsets otherwise, so one large polygon costs only
  // its own rows)
  std::vector<uint32_t> rec(npoly);
  uint64_t units = 0, umax = 0;
  for (uint32_t i = 0; i < npoly; ++i) {
    rec[i] = static_cast<uint32_t>(units);
    const uint64_t nn = offsets[i + 1] - offsets[i];
    const uint64_t u = 1 + std::max<uint64_t>(2, (nn + 3) / 4);  // header, >= two 4-row chunks
    units += u;
    umax = std::max(umax, u);
  }
  uint32_t stride = 0;
  if (npoly && umax * npoly <= units + units / 2 && umax <= 1024) {
    stride = static_cast<uint32_t>(umax);
    units = umax * npoly;
    for (uint32_t i = 0; i < npoly; ++i) rec[i] = i * stride;
  }
  if (units > UINT32_MAX) {  // record offsets are u32 in 32-byte units (128 GiB)
    delete db;
    return kInvalid;
  }
  size_t off = 0;
  auto take = [&](size_t bytes) { const size_t o = off; off = align256(off + bytes); return o; };
  const size_t o_offs = take((npoly + 1) * sizeof(uint32_t));
  const size_t o_rec = take(npoly * sizeof(uint32_t));
  const size_t o_vx = take(nv * sizeof(double)), o_vy = take(nv * sizeof(double));
  const size_t o_inner = take(npoly * sizeof(double2)), o_outer = take(nv * sizeof(double2));
  const size_t o_recs = take(units * 32);
  const size_t o_status = take(npoly * sizeof(int32_t));
  // stream-ordered allocation from the library's per-device pool (warm ingest
  // pays no cudaMalloc), released stream-ordered by vpipg_db_destroy
  cudaMemPool_t pool = nullptr;
  rc = blob_pool(device, &pool);
  if (rc) {
    delete db;
    return rc;
  }
  cudaError_t e = cudaMallocFromPoolAsync(&db->blob, off ? off : 256, pool, s);
  if (e != cudaSuccess) {
    delete db;
    return cuda_code(e);
  }
  char* b = static_cast<char*>(db->blob);
  CsrPrepArgs a{};
  a.offsets = reinterpret_cast<const uint32_t*>(b + o_offs);
  a.rec = reinterpret_cast<const uint32_t*>(b + o_rec);
  a.vx = reinterpret_cast<const double*>(b + o_vx);
  a.vy = reinterpret_cast<const double*>(b + o_vy);
  a.npoly = npoly;
  a.kinds = kinds;
  a.inner = reinterpret_cast<double2*>(b + o_inner);
  a.outer = reinterpret_cast<double2*>(b + o_outer);
  a.recs = reinterpret_cast<float2*>(b + o_recs);
  a.status = reinterpret_cast<int32_t*>(b + o_status);
  std::vector<int32_t> status(npoly);
  do {
    // the generators of polygons that fail validation read back as zeros
    if ((e = cudaMemsetAsync(b + o_inner, 0, o_recs - o_inner, s)) != cudaSuccess) break;
    if ((e = cudaMemcpyAsync(b + o_offs, offsets, (npoly + 1) * sizeof(uint32_t), cudaMemcpyHostToDevice, s)) != cudaSuccess) break;
    if (npoly && (e = cudaMemcpyAsync(b + o_rec, rec.data(), npoly * sizeof(uint32_t), cudaMemcpyHostToDevice, s)) != cudaSuccess) break;
    if (nv && (e = cudaMemcpyAsync(b + o_vx, vx, nv * sizeof(double), cudaMemcpyHostToDevice, s)) != cudaSuccess) break;
    if (nv && (e = cudaMemcpyAsync(b + o_vy, vy, nv * sizeof(double), cudaMemcpyHostToDevice, s)) != cudaSuccess) break;
    if ((e = launch_prep_csr(a, s)) != cudaSuccess) break;
    if (npoly && (e = cudaMemcpyAsync(status.data(), a.status, npoly * sizeof(int32_t), cudaMemcpyDeviceToHost, s)) != cudaSuccess) break;
    e = cudaStreamSynchronize(s);
  } while (false);
  if (e != cudaSuccess) {
    vpipg_db_destroy(db);
    return cuda_code(e);
  }
  if (per_poly_status) std::copy(status.begin(), status.end(), per_poly_status);
  db->t = DbTables{npoly, kinds, stride, a.rec, a.recs};
  db->d_offsets = a.offsets;
  db->d_inner = a.inner;
  db->d_outer = a.outer;
  *out = db;
  return kOk;
}

void vpipg_db_destroy(vpipg_db* db) {
  if (!db) return;
  if (db->blob) {
    DeviceGuard g(db->device);
    cudaFreeAsync(db->blob, nullptr);  // back to the pool, as vpipg_destroy
  }
  delete db;
}

int vpipg_db_info(const vpipg_db* db, uint32_t* npoly, uint64_t* nverts, uint32_t* kinds) {
  if (!db) return kInvalid;
  if (npoly) *npoly = db->npoly;
  if (nverts) *nverts = db->nverts;
  if (kinds) *kinds = db->kinds;
  return kOk;
}

int vpipg_db_generators(const vpipg_db* db, uint32_t poly, double* inner_xy, double* outer_xy) {
  if (!db || !(db->kinds & kKindVoronoi) || poly >= db->npoly || !inner_xy) return kInvalid;
  const uint32_t s = db->offsets[poly], n = db->offsets[poly + 1] - s;
  if (n && !outer_xy) return kInvalid;
  DeviceGuard g(db->device);
  VPIPG_TRY(cudaMemcpy(inner_xy, db->d_inner + poly, sizeof(double2), cudaMemcpyDeviceToHost));
  if (n) VPIPG_TRY(cudaMemcpy(outer_xy, db->d_outer + s, n * sizeof(double2), cudaMemcpyDeviceToHost));
  return kOk;
}

int vpipg_test_gather(const vpipg_db* db, int engine, const float* xs, const float* ys,
                      const uint32_t* ids, uint64_t m, uint32_t* mask_words, uint8_t* mask_bytes,
                      unsigned long long* d_inside, void* stream) {
  if (!db || engine < 0 || engine > 2) return kInvalid;
  const uint32_t need = engine == 0 ? kKindVoronoi : engine == 1 ? kKindOffset : kKindCrossing;
  if (!(db->kinds & need)) return kInvalid;
  if (m == 0) return kOk;
  if (!xs || !ys || !ids) return kInvalid;
  DeviceGuard g(db->device);
  GatherArgs a{xs, ys, ids, m, mask_words, mask_bytes, d_inside};
  return cuda_code(launch_gather(db->t, engine, a, static_cast<cudaStream_t>(stream)));
}

int vpipg_test_gather_multi(const vpipg_db* db, uint32_t engines, const float* xs, const float* ys,
                            const uint32_t* ids, uint64_t m, uint32_t* const* mask_words,
                            uint8_t* const* mask_bytes, unsigned long long* const* d_inside,
                            void* stream) {
  if (!db || engines == 0 || (engines & ~7u)) return kInvalid;
  for (int e = 0; e < 3; ++e) {
    const uint32_t need = e == 0 ? kKindVoronoi : e == 1 ? kKindOffset : kKindCrossing;
    if ((engines & (1u << e)) && !(db->kinds & need)) return kInvalid;
  }
  if (m == 0) return kOk;
  if (!xs || !ys || !ids) return kInvalid;
  DeviceGuard g(db->device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  GatherArgs a[3];
  for (int e = 0; e < 3; ++e)
    a[e] = GatherArgs{xs, ys, ids, m, mask_words ? mask_words[e] : nullptr,
                      mask_bytes ? mask_bytes[e] : nullptr, d_inside ? d_inside[e] : nullptr};
  if (engines == 7u) return cuda_code(launch_gather_all(db->t, a, s));
  for (int e = 0; e < 3; ++e)
    if (engines & (1u << e)) {
      const int rc = cuda_code(launch_gather(db->t, e, a[e], s));
      if (rc) return rc;
    }
  return kOk;
}

int vpipg_fill_join_pairs(uint64_t seed, uint64_t first, uint64_t m, uint32_t npoly,
                          const double* centre_x, const double* centre_y, const double* radius,
                          float* xs, float* ys, uint32_t* ids, void* stream) {
  if (m && (npoly == 0 || !centre_x || !centre_y || !radius || !xs || !ys || !ids)) return kInvalid;
  return cuda_code(launch_fill_pairs(seed, first, m, npoly, centre_x, centre_y, radius, xs, ys,
                                     ids, static_cast<cudaStream_t>(stream)));
}

namespace {

double poly_extent(const vpipg_poly* p) {
  if (p->vx.empty()) return 0.0;
  const auto [x0, x1] = std::minmax_element(p->vx.begin(), p->vx.end());
  const auto [y0, y1] = std::minmax_element(p->vy.begin(), p->vy.end());
  return std::max(*x1 - *x0, *y1 - *y0);
}

int classify(const vpipg_poly* p, int dtype, const void* xs, const void* ys, uint64_t m,
             const uint32_t* w0, const uint32_t* w1, const uint32_t* w2, double band,
             int relative, vpipg_report* out, cudaStream_t s) {
  ReportDev* rep = nullptr;
  VPIPG_TRY(cudaMallocAsync(reinterpret_cast<void**>(&rep), sizeof(ReportDev), s));
  int rc = kOk;
  auto fail = [&](cudaError_t e) {
    if (e != cudaSuccess && rc == kOk) rc = cuda_code(e);
    return rc != kOk;
  };
  if (const int st = ensure_ready(p)) return st;
  ClassifyArgs a{{w0, w1, w2}, xs, ys, dtype, m, band, relative, poly_extent(p), p->t.lines,
                 p->n, rep};
  // counters only (the sample arrays are written before they are read)
  struct Head {
    unsigned long long pair[3], dis, out, rec;
  } head{};
  std::vector<unsigned long long> idx;
  std::vector<double> dist;
  std::vector<uint32_t> bits;
  if (!fail(cudaMemsetAsync(rep, 0, sizeof(Head), s)) && !fail(launch_classify(a, s)) &&
      !fail(cudaMemcpyAsync(&head, rep, sizeof(Head), cudaMemcpyDeviceToHost, s)) &&
      !fail(cudaStreamSynchronize(s))) {
    const size_t k = std::min<unsigned long long>(head.rec, kSampleCapacity);
    idx.resize(k);
    dist.resize(k);
    bits.resize(k);
    if (k) {
      fail(cudaMemcpyAsync(idx.data(), rep->sample_index, k * 8, cudaMemcpyDeviceToHost, s));
      fail(cudaMemcpyAsync(dist.data(), rep->sample_dist, k * 8, cudaMemcpyDeviceToHost, s));
      fail(cudaMemcpyAsync(bits.data(), rep->sample_bits, k * 4, cudaMemcpyDeviceToHost, s));
      fail(cudaStreamSynchronize(s));
    }
  }
  cudaFreeAsync(rep, s);
  if (rc) return rc;
  std::memset(out, 0, sizeof(*out));
  out->point_count = m;
  for (int i = 0; i < 3; ++i) out->pair_disagreements[i] = head.pair[i];
  if (!w2) out->pair_disagreements[2] = 0;
  out->disagreeing_points = head.dis;
  out->outside_band = head.out;
  out->pass = head.out == 0;
  // the first disagreements by index (exact while fewer than kSampleCapacity occurred)
  std::vector<size_t> order(idx.size());
  for (size_t i = 0; i < order.size(); ++i) order[i] = i;
  std::sort(order.begin(), order.end(), [&](size_t a1, size_t b1) { return idx[a1] < idx[b1]; });
  out->n_samples = static_cast<uint32_t>(std::min<size_t>(order.size(), VPIPG_REPORT_SAMPLES));
  for (uint32_t i = 0; i < out->n_samples; ++i) {
    out->sample_index[i] = idx[order[i]];
    out->sample_dist[i] = dist[order[i]];
    out->sample_engines[i] = bits[order[i]];
  }
  return kOk;
}

}  // namespace

int vpipg_validate(const vpipg_poly* p, int dtype, const void* xs, const void* ys, uint64_t m,
                   double band, int band_relative, vpipg_report* out, void* stream) {
  if (!p || !out || (p->kinds & VPIPG_KIND_ALL) != VPIPG_KIND_ALL) return kInvalid;
  if (dtype != VPIPG_F32 && dtype != VPIPG_F64) return kInvalid;
  if (m && (!xs || !ys)) return kInvalid;
  DeviceGuard g(p->device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const uint64_t nw = (m + 31) / 32;
  uint32_t* w = nullptr;
  VPIPG_TRY(cudaMallocAsync(reinterpret_cast<void**>(&w), 3 * std::max<uint64_t>(nw, 1) * 4, s));
  int rc = kOk;
  for (int e = 0; e < 3 && rc == kOk; ++e) {
    TestArgs a{xs, ys, m, w + e * nw, nullptr, nullptr};
    rc = dispatch(p, e, dtype, a, s);
  }
  if (rc == kOk) rc = classify(p, dtype, xs, ys, m, w, w + nw, w + 2 * nw, band, band_relative, out, s);
  cudaFreeAsync(w, s);
  cudaStreamSynchronize(s);
  return rc;
}

int vpipg_compare_masks(const vpipg_poly* p, int dtype, const void* xs, const void* ys,
                        uint64_t m, const uint32_t* words_a, const uint32_t* words_b, double band,
                        int band_relative, vpipg_report* out, void* stream) {
  if (!p || !out || (m && (!xs || !ys || !words_a || !words_b))) return kInvalid;
  if (dtype != VPIPG_F32 && dtype != VPIPG_F64) return kInvalid;
  DeviceGuard g(p->device);
  return classify(p, dtype, xs, ys, m, words_a, words_b, nullptr, band, band_relative, out,
                  static_cast<cudaStream_t>(stream));
}

int vpipg_voronoi_work(const vpipg_poly* p, uint64_t m, uint64_t* evals, uint64_t* comps) {
  if (!p || !(p->kinds & kKindVoronoi)) return kInvalid;
  if (evals) *evals = (uint64_t(p->n) + 1) * m;
  if (comps) *comps = uint64_t(p->n) * m;
  return kOk;
}

int vpipg_fill_uniform_points(uint64_t seed, uint64_t first, uint64_t m, double min_x,
                              double min_y, double max_x, double max_y, int dtype, void* xs,
                              void* ys, void* stream) {
  if ((dtype != VPIPG_F32 && dtype != VPIPG_F64) || (m && (!xs || !ys))) return kInvalid;
  if (!(min_x < max_x && min_y < max_y)) return kInvalid;
  return cuda_code(launch_fill_uniform(seed, first, m, min_x, min_y, max_x, max_y, dtype, xs, ys,
                                       static_cast<cudaStream_t>(stream)));
}

}  // extern "C"

namespace vpipg {

cudaError_t launch_config(const void* kernel, int threads, size_t smem, int* sms, int* per_sm) {
  struct Key {
    int dev;
    const void* k;
    int threads;
    size_t smem;
    bool operator<(const Key& o) const {
      return std::tie(dev, k, threads, smem) < std::tie(o.dev, o.k, o.threads, o.smem);
    }
  };
  static std::mutex mu;
  static std::map<Key, std::pair<int, int>> cache;              // -> (sms, blocks per SM)
  static std::map<std::pair<int, const void*>, size_t> smem_set;  // largest limit set so far
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lock(mu);
  const Key key{dev, kernel, threads, smem};
  const auto hit = cache.find(key);
  if (hit != cache.end()) {
    *sms = hit->second.first;
    *per_sm = hit->second.second;
    return cudaSuccess;
  }
  size_t& lim = smem_set[{dev, kernel}];
  if (smem > 48 * 1024 && smem > lim) {
    e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    lim = smem;
  }
  int n = 0, b = 0;
  if ((e = cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev)) != cudaSuccess) return e;
  if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, kernel, threads, smem)) != cudaSuccess)
    return e;
  b = b < 1 ? 1 : b;
  cache[key] = {n, b};
  *sms = n;
  *per_sm = b;
  return cudaSuccess;
}

}  // namespace vpipg
