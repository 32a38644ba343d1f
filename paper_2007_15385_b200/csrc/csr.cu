// csr.cu -- polygon-database join (BASELINE config 4): batched device
// preparation of a CSR polygon table and the gather test kernels.
//
// prep_csr_kernel, one thread per polygon:
//   validate_polygon (geometry.cpp:53-98) -> per-polygon status, CCW order,
//   to_voronoi (voronoi.cpp:60-71) with the reference's exact f64 arithmetic,
//   then fp32 half-plane tables in affine form a*x + b*y + c >= 0 (unit
//   normal, so the value is a signed distance) for the Voronoi engine (from
//   the generators: perpendicular bisector of inner and outer[k]) and the
//   sign-of-offset engine (from the edges, engines.cpp:146-152), and the
//   crossing table (x, y, dvx/dvy) from the RAW vertices (vpip.cpp:120-128).
// gather_kernel: every (point, polygon id) pair fetches its own polygon's
//   rows from the L2-resident tables (per-lane loops of divergent length),
//   2 FFMA + 1/2 LOP3 per point-edge for the affine engines, the test_f32.cu
//   crossing arithmetic for ray crossing; ballot words, fused counts.
#include <climits>
#include <cmath>
#include <cstdint>

#include "exact_geom.cuh"
#include "vpipg_device.cuh"
#include "vpipg_internal.h"

namespace vpipg {

namespace {

struct CsrView {
  const double* x;
  const double* y;
  __device__ double2 operator()(int k) const { return make_double2(x[k], y[k]); }
};

__device__ float4 unit_halfplane(double a, double b, double c) {
  const double s = 1.0 / hypot(a, b);
  return make_float4(static_cast<float>(a * s), static_cast<float>(b * s),
                     static_cast<float>(c * s), 0.f);
}

__global__ void prep_csr_kernel(CsrPrepArgs a) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= a.npoly) return;
  const uint32_t s = a.offsets[i];
  const int n = static_cast<int>(a.offsets[i + 1] - s);
  const CsrView raw{a.vx + s, a.vy + s};
  int status = 0;
  bool rev = false;
  const bool convex = a.kinds & (kKindVoronoi | kKindOffset);
  if (convex) status = validate_exact(raw, n, &rev);
  double* vvx = a.vvx + s;
  double* vvy = a.vvy + s;
  for (int k = 0; k < n; ++k) {
    const double2 p = raw(rev ? n - 1 - k : k);
    vvx[k] = p.x;
    vvy[k] = p.y;
  }
  const CsrView val{vvx, vvy};
  if (status == 0 && (a.kinds & kKindVoronoi)) {
    double cx, cy;
    centroid_exact(val, n, &cx, &cy);
    a.inner[i] = make_double2(cx, cy);
    for (int k = 0; k < n && status == 0; ++k) {
      double2 g;
      status = reflect_exact(val(k), val((k + 1) % n), cx, cy, &g);
      if (status) break;
      a.outer[s + k] = g;
      // |x - p0|^2 <= |x - pk|^2  <=>  d.(m - x) >= 0, d = pk - p0, m = midpoint
      const double dx = g.x - cx, dy = g.y - cy;
      const double mx = 0.5 * (cx + g.x), my = 0.5 * (cy + g.y);
      a.vor[s + k] = unit_halfplane(-dx, -dy, dx * mx + dy * my);
    }
  }
  if (status == 0 && (a.kinds & kKindOffset)) {
    for (int e = 0; e < n; ++e) {
      const double2 u = val(e), w = val((e + n - 1) % n);
      const double dvx = u.x - w.x, dvy = u.y - w.y;
      a.off[s + e] = unit_halfplane(-dvy, dvx, w.x * dvy - w.y * dvx);
    }
  }
  if (a.kinds & kKindCrossing) {
    for (int k = 0; k < n; ++k) {
      const double2 u = raw(k), w = raw((k + n - 1) % n);
      const double dvy = u.y - w.y;
      a.cross[s + k] = make_float4(static_cast<float>(u.x), static_cast<float>(u.y),
                                   dvy != 0.0 ? static_cast<float>((u.x - w.x) / dvy) : 0.f, 0.f);
    }
  }
  a.status[i] = status;
  // a failed polygon tests outside under Voronoi / sign-of-offset (crossing
  // ignores the flag: it accepts any polygon)
  const bool bad = convex && status != 0;
  a.range[i] = make_uint2(s, static_cast<uint32_t>(n) | (bad ? kRangeInvalid : 0u));
}

constexpr int kGP = 4;  // pairs per lane
constexpr int kGThreads = 256;

template <int kEngine>  // 0 voronoi, 1 offset: affine tables; 2 crossing
__global__ void __launch_bounds__(kGThreads) gather_kernel(const DbTables t, const GatherArgs a) {
  const int lane = threadIdx.x & 31;
  const uint64_t gwarp = (uint64_t)blockIdx.x * (kGThreads / 32) + (threadIdx.x >> 5);
  const uint64_t stride = (uint64_t)gridDim.x * (kGThreads / 32) * 32 * kGP;
  const float4* rows = kEngine == 0 ? t.vor : kEngine == 1 ? t.off : t.cross;
  uint32_t count = 0;
  for (uint64_t base = gwarp * 32 * kGP; base < a.m; base += stride) {
    float x[kGP], y[kGP];
    uint32_t start[kGP], n[kGP];
    bool ok[kGP];
    uint32_t nmax = 0;
#pragma unroll
    for (int p = 0; p < kGP; ++p) {
      const uint64_t j = base + 32u * p + lane;
      ok[p] = j < a.m;
      const uint32_t id = ok[p] ? __ldcs(a.ids + j) : 0u;
      x[p] = ok[p] ? __ldcs(a.xs + j) : 0.f;
      y[p] = ok[p] ? __ldcs(a.ys + j) : 0.f;
      ok[p] = ok[p] && id < t.npoly;
      const uint2 r = ok[p] ? __ldg(t.range + id) : make_uint2(0u, 0u);
      // a polygon that failed validation only disables the convex engines: ray
      // crossing takes the raw vertices of any polygon (vpip.cpp:120-128)
      if (kEngine != 2) ok[p] = ok[p] && !(r.y & kRangeInvalid);
      start[p] = r.x;
      n[p] = ok[p] ? (r.y & ~kRangeInvalid) : 0u;
      nmax = n[p] > nmax ? n[p] : nmax;
    }
    bool in[kGP];
    if (kEngine != 2) {
      uint32_t acc[kGP];
#pragma unroll
      for (int p = 0; p < kGP; ++p) acc[p] = 0;
      for (uint32_t e = 0; e < nmax; ++e) {
#pragma unroll
        for (int p = 0; p < kGP; ++p) {
          if (e < n[p]) {
            const float4 c = __ldg(rows + start[p] + e);
            acc[p] |= __float_as_uint(fmaf(c.x, x[p], fmaf(c.y, y[p], c.z)));
          }
        }
      }
#pragma unroll
      for (int p = 0; p < kGP; ++p) in[p] = ok[p] && !(acc[p] >> 31);
    } else {
      uint32_t par[kGP];
      float hp[kGP], gp[kGP];
#pragma unroll
      for (int p = 0; p < kGP; ++p) {
        par[p] = 0;
        const float4 last = n[p] ? __ldg(rows + start[p] + n[p] - 1) : make_float4(0.f, 0.f, 0.f, 0.f);
        hp[p] = y[p] - last.y;
        gp[p] = last.x - x[p];
      }
      for (uint32_t k = 0; k < nmax; ++k) {
#pragma unroll
        for (int p = 0; p < kGP; ++p) {
          if (k < n[p]) {
            const float4 v = __ldg(rows + start[p] + k);
            const float h = y[p] - v.y;
            const float d = fmaf(hp[p], v.z, gp[p]);
            par[p] ^= (__float_as_uint(h) ^ __float_as_uint(hp[p])) & ~__float_as_uint(d);
            hp[p] = h;
            gp[p] = v.x - x[p];
          }
        }
      }
#pragma unroll
      for (int p = 0; p < kGP; ++p) in[p] = ok[p] && (par[p] >> 31);
    }
    uint32_t w[kGP];
#pragma unroll
    for (int p = 0; p < kGP; ++p) {
      w[p] = __ballot_sync(0xffffffffu, in[p]);
      count += in[p];
    }
    if (a.words && lane == 0) {
      const uint64_t w0 = base >> 5, nwords = (a.m + 31) >> 5;
#pragma unroll
      for (int p = 0; p < kGP; ++p)
        if (w0 + p < nwords) a.words[w0 + p] = w[p];
    }
    if (a.bytes) {
#pragma unroll
      for (int p = 0; p < kGP; ++p) {
        const uint64_t j = base + 32u * p + lane;
        if (j < a.m) a.bytes[j] = in[p] ? 1 : 0;
      }
    }
  }
#pragma unroll
  for (int s = 16; s > 0; s >>= 1) count += __shfl_xor_sync(0xffffffffu, count, s);
  if (lane == 0 && a.inside && count) atomicAdd(a.inside, (unsigned long long)count);
}

__device__ __forceinline__ uint64_t mix_seed(uint64_t seed, uint64_t salt) {
  uint64_t z = seed + 0x9e3779b97f4a7c15ULL * (salt + 1);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

__device__ __forceinline__ double unit(uint64_t r) {
  return __dmul_rn(static_cast<double>(r >> 11), 0x1.0p-53);
}

// Join pairs: id = floor(U(seed, 3j) * npoly), point = centre + (2U - 1) * r per
// axis (a 2r x 2r box around the polygon centre), rounded once to f32.
__global__ void fill_pairs_kernel(uint64_t seed, uint64_t first, uint64_t m, uint32_t npoly,
                                  const double* cx, const double* cy, const double* rad,
                                  float* xs, float* ys, uint32_t* ids) {
  for (uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; t < m;
       t += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t j = first + t;
    uint32_t id = static_cast<uint32_t>(__dmul_rn(unit(mix_seed(seed, 3 * j)), (double)npoly));
    if (id >= npoly) id = npoly - 1;
    const double r = rad[id];
    const double ux = __dsub_rn(__dmul_rn(2.0, unit(mix_seed(seed, 3 * j + 1))), 1.0);
    const double uy = __dsub_rn(__dmul_rn(2.0, unit(mix_seed(seed, 3 * j + 2))), 1.0);
    xs[t] = static_cast<float>(__dadd_rn(cx[id], __dmul_rn(ux, r)));
    ys[t] = static_cast<float>(__dadd_rn(cy[id], __dmul_rn(uy, r)));
    ids[t] = id;
  }
}

}  // namespace

cudaError_t launch_prep_csr(const CsrPrepArgs& a, cudaStream_t stream) {
  if (a.npoly == 0) return cudaSuccess;
  prep_csr_kernel<<<(a.npoly + 127) / 128, 128, 0, stream>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_gather(const DbTables& t, int engine, const GatherArgs& a, cudaStream_t stream) {
  if (a.m == 0) return cudaSuccess;
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const uint64_t warps = (a.m + 32 * kGP - 1) / (32 * kGP);
  const uint64_t blocks = (warps + kGThreads / 32 - 1) / (kGThreads / 32);
  const uint64_t cap = (uint64_t)sms * 8;
  const int grid = static_cast<int>(blocks < cap ? blocks : cap);
  switch (engine) {
    case 0: gather_kernel<0><<<grid, kGThreads, 0, stream>>>(t, a); break;
    case 1: gather_kernel<1><<<grid, kGThreads, 0, stream>>>(t, a); break;
    default: gather_kernel<2><<<grid, kGThreads, 0, stream>>>(t, a); break;
  }
  return cudaGetLastError();
}

cudaError_t launch_fill_pairs(uint64_t seed, uint64_t first, uint64_t m, uint32_t npoly,
                              const double* cx, const double* cy, const double* rad, float* xs,
                              float* ys, uint32_t* ids, cudaStream_t stream) {
  if (m == 0) return cudaSuccess;
  const uint64_t blocks64 = (m + 255) / 256;
  const int blocks = static_cast<int>(blocks64 < 148 * 64 ? blocks64 : 148 * 64);
  fill_pairs_kernel<<<blocks, 256, 0, stream>>>(seed, first, m, npoly, cx, cy, rad, xs, ys, ids);
  return cudaGetLastError();
}

}  // namespace vpipg
