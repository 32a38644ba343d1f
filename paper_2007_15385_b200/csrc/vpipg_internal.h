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
  PrepMeta* meta;
};

struct TestArgs {
  const void* xs;
  const void* ys;
  uint64_t m;
  uint32_t* words;
  uint8_t* bytes;
  unsigned long long* inside;
};

cudaError_t launch_prep(const PrepArgs& args, cudaStream_t stream);
cudaError_t launch_test_f32(const DevTables& t, int engine, const TestArgs& a, cudaStream_t stream);
cudaError_t launch_test_f64(const DevTables& t, int engine, const TestArgs& a, cudaStream_t stream);
cudaError_t launch_fill_uniform(uint64_t seed, uint64_t first, uint64_t m, double min_x,
                                double min_y, double max_x, double max_y, int dtype, void* xs,
                                void* ys, cudaStream_t stream);

}  // namespace vpipg
