// capi_internal.h -- state and helpers shared by the host-side C-ABI
// translation units (capi.cu: handles, prepare, device-buffer calls,
// validation; hostpipe.cu: the host-buffer pipelines).
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <cstddef>
#include <cstdint>
#include <mutex>
#include <vector>

#include "vpipg.h"
#include "vpipg_internal.h"

// A prepared polygon. vpipg_prepare only enqueues the device conversion
// (upload, prep kernel, download of the status / slab counts / f32 tables into
// pinned host memory, an event) and returns; the first call that needs the
// results waits for the event and finishes the handle (capi::ensure_ready),
// once, under `mu`. Finished handles are immutable.
struct vpipg_poly {
  int device = 0;
  uint32_t n = 0;
  uint32_t kinds = 0;
  int reversed = 0;
  void* blob = nullptr;
  std::vector<double> vx, vy;  // validated (or raw, crossing-only) vertices
  // ---- asynchronous preparation ----
  cudaEvent_t ready = nullptr;   // recorded after the download
  char* host = nullptr;          // pinned block: uploads, then the download
  size_t host_bytes = 0;
  size_t dl_meta = 0;            // offsets in `host` of the downloaded
  size_t dl_slab[2] = {0, 0};    //   PrepMeta, slab tables and crossing table
  size_t dl_cross = 0;
  bool host_tables = false;      // the f32 tables were downloaded (n small)
  vpipg::PrepArgs args{};        // device table pointers (into blob)
  mutable std::mutex mu;
  mutable std::atomic<int> state{-1};  // -1 pending, 0 ready, > 0 the prep error code
  mutable vpipg::DevTables t{};
  mutable double inner_x = 0, inner_y = 0;
};

struct vpipg_db {
  int device = 0;
  uint32_t npoly = 0;
  uint64_t nverts = 0;
  uint32_t kinds = 0;
  void* blob = nullptr;
  vpipg::DbTables t{};
  const uint32_t* d_offsets = nullptr;
  const double2* d_inner = nullptr;
  const double2* d_outer = nullptr;
  std::vector<uint32_t> offsets;
};

namespace vpipg::capi {

constexpr int kOk = 0;
constexpr int kTooFew = 1, kNotConvex = 2, kDegenerate = 3, kNonFinite = 4;
constexpr int kInvalid = 6;

inline int cuda_code(cudaError_t e) {
  return e == cudaSuccess ? kOk : VPIPG_ERR_CUDA + static_cast<int>(e);
}

inline size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

#define VPIPG_TRY(expr)                                       \
  do {                                                        \
    const cudaError_t e_ = (expr);                            \
    if (e_ != cudaSuccess) return ::vpipg::capi::cuda_code(e_); \
  } while (0)

// Sets the polygon's device for the scope of a call, restores the caller's.
struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

// Waits for a handle's asynchronous preparation (once) and fills its tables;
// 0 or the prep kernel's error code (capi.cu).
int ensure_ready(const vpipg_poly* p);

// Launches engine `engine` of a prepared polygon on device buffers (capi.cu).
int dispatch(const vpipg_poly* p, int engine, int dtype, const TestArgs& a, cudaStream_t s);

}  // namespace vpipg::capi
