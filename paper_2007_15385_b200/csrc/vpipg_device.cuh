// vpipg_device.cuh -- device-side table layout shared by the prep and test
// kernels of the B200 point-inclusion engine.
//
// A prepared polygon lives in ONE device allocation (the "blob") holding:
//   exact f64 tables  -- the reference's own operands, so the f64 kernels
//                        repeat its arithmetic bit for bit:
//                        Voronoi generators (voronoi.hpp:58-65), per-edge
//                        (dvx, dvy, rhs) of the sign-of-offset kernel
//                        (engines.cpp:146-149) and the ray-crossing edge
//                        record (engines.cpp:177-186);
//   fp32 affine tables -- per-edge comparison coefficients in a polygon-local
//                        frame (origin o = f32(centroid)), in "slab" form:
//                        each half-plane a*x' + b*y' + c >= 0 is divided by
//                        its larger |coefficient| and becomes one of
//                          x' >= B*y' + C (XLO), x' <= B*y' + C (XHI),
//                          y' >= B*x' + C (YLO), y' <= B*x' + C (YHI),
//                        with |B| <= 1. A point is inside iff
//                        max(XLO) <= x' <= min(XHI) and max(YLO) <= y' <= min(YHI):
//                        one FFMA per point-edge plus half an FMNMX3.
#pragma once

#include <cstdint>

namespace vpipg {

constexpr int kGroups = 4;  // XLO, XHI, YLO, YHI

// One engine's fp32 half-plane set. Groups are stored back to back in
// `coef` as (B, C) pairs; each group is padded to an even length with a
// neutral entry (C = -inf for max groups, +inf for min groups) so the
// kernels consume two edges per 16-byte load.
struct SlabTable {
  const float2* coef;
  uint32_t off[kGroups];
  uint32_t cnt[kGroups];
  uint32_t total;  // sum of cnt
  uint32_t pad_;
};

// Ray-crossing fp32 table: per vertex k, (x'_k, y'_k, B_k, 0) with
// B_k = dvx/dvy of the edge v[k-1] -> v[k] (0 for horizontal edges, which
// are never in range). Vertices are local-frame f32.
struct CrossTable {
  const float4* vert;
  uint32_t n;
  uint32_t pad_;
};

struct OffsetEdgeF64 {  // engines.cpp:147-149, edge j -> i with i = e, j = e-1
  double dvx, dvy, rhs, pad_;
};

struct RayEdgeF64 {  // engines.cpp:177-186, edge w = v[j] -> u = v[i]
  double wy, uy, dvx, dvy, rhs, min_x, max_x, min_y, max_y;
  int going_up;
  int pad_;
};

// Kernel parameter block (passed by value; points into the blob).
struct DevTables {
  uint32_t n;
  uint32_t kinds;
  // f64 exact
  double inner_x, inner_y;
  const double2* outer;      // n generators
  const OffsetEdgeF64* off;  // n
  const RayEdgeF64* ray;     // n
  // f32 affine
  float ox, oy;              // local-frame origin (f32 centroid; a zero coordinate is +0.0f)
  SlabTable slab[2];         // [0] Voronoi (from generators), [1] sign-of-offset
  CrossTable cross;
  // unit-normal supporting lines (a, b, c, 0) of the n edges, f64: the band
  // metric edge_line_distance (voronoi.cpp:73-82) of the validation kernels
  const double4* lines;
  // host copies of the f32 tables (slab (B, C) pairs, crossing records) for
  // launches that pass them in the kernel parameter bank; null when absent
  const float2* h_slab[2];
  const float4* h_cross;
};

// Written by the prep kernel, read back by the (synchronous) prepare call.
struct PrepMeta {
  int status;                 // 0 or vpip::ErrorCode + 1
  uint32_t cnt[2][kGroups];   // padded slab group sizes per engine
  double inner_x, inner_y;    // the generator (centroid) actually used
  float ox, oy;
};

}  // namespace vpipg
