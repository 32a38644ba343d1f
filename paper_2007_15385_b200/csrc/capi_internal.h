// capi_internal.h -- state and helpers shared by the host-side C-ABI
// translation units (capi.cu: handles, prepare, device-buffer calls,
// validation; hostpipe.cu: the host-buffer pipelines).
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>
#include <vector>

#include "vpipg.h"
#include "vpipg_internal.h"

struct vpipg_poly {
  int device = 0;
  uint32_t n = 0;
  uint32_t kinds = 0;
  int reversed = 0;
  void* blob = nullptr;
  vpipg::DevTables t{};
  std::vector<double> vx, vy;  // validated (or raw, crossing-only) vertices
  double inner_x = 0, inner_y = 0;
  std::vector<float2> h_slab[2];  // host copies of the f32 tables (DevTables::h_*)
  std::vector<float4> h_cross;
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

// Launches engine `engine` of a prepared polygon on device buffers (capi.cu).
int dispatch(const vpipg_poly* p, int engine, int dtype, const TestArgs& a, cudaStream_t s);

}  // namespace vpipg::capi
