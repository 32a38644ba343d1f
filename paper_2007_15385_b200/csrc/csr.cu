// csr.cu -- polygon-database join (BASELINE config 4): batched device
// preparation of a CSR polygon table and the gather test kernels.
//
// prep_csr_kernel, one thread per polygon:
//   validate_polygon (geometry.cpp:53-98) -> per-polygon status, CCW order,
//   to_voronoi (voronoi.cpp:60-71) with the reference's exact f64 arithmetic,
//   then one fixed-stride, 32-byte-aligned block per polygon and engine: a
//   16-byte header (n | invalid flag, frame origin c) and fp32 rows in the
//   polygon-local frame: the n outer generators (Voronoi, c = the centroid
//   rounded to f32, so the inner generator is the origin), the validated
//   vertices (sign-of-offset) and the RAW vertices (ray crossing,
//   vpip.cpp:120-128), both as v_{n-1}, v_0 .. v_{n-1} with c = the f32
//   bounding-box centre.
// gather_kernel: every (point, polygon id) pair reads its polygon's block in
//   32-byte loads (header + 2 rows, then 4 rows at a time) from the
//   L2-resident tables; q' = q - c is exact in f32 (Sterbenz) for points near
//   their polygon. Per point-edge:
//     Voronoi    |q'-pk'|^2 - |q'-p0'|^2 >= 0 (the reference's squared
//                distances, engines.cpp:85-98): 5 FP ops
//     offset     a_j*b_i - a_i*b_j >= 0 with (a, b) = q' - v': the cross
//                product (q - v_j) x (v_i - v_j) of engines.cpp:150-152
//     crossing   in_range = H_i ^ H_j, on_left = sign(s) ^ H_i (H = [v.y > qy],
//                s the same cross product), parity by XOR (engines.cpp:187-196)
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

__device__ __forceinline__ float2 local(double2 p, double cx, double cy) {
  return make_float2(static_cast<float>(p.x - cx), static_cast<float>(p.y - cy));
}

__global__ void prep_csr_kernel(CsrPrepArgs a) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= a.npoly) return;
  const uint32_t s = a.offsets[i];
  const int n = static_cast<int>(a.offsets[i + 1] - s);
  const uint64_t blk = (uint64_t)i * a.stride;
  const CsrView raw{a.vx + s, a.vy + s};
  int status = 0;
  bool rev = false;
  const bool convex = a.kinds & (kKindVoronoi | kKindOffset);
  if (convex) status = validate_exact(raw, n, &rev);
  double* vvx = a.vvx + s;
  double* vvy = a.vvy + s;
  double x0 = INFINITY, x1 = -INFINITY, y0 = INFINITY, y1 = -INFINITY;
  for (int k = 0; k < n; ++k) {
    const double2 p = raw(rev ? n - 1 - k : k);
    vvx[k] = p.x;
    vvy[k] = p.y;
    if (isfinite(p.x) && isfinite(p.y)) {
      x0 = fmin(x0, p.x); x1 = fmax(x1, p.x);
      y0 = fmin(y0, p.y); y1 = fmax(y1, p.y);
    }
  }
  // polygon-local frame: f32 centre of the bounding box (exactly representable)
  const float fcx = (x0 <= x1) ? static_cast<float>(0.5 * (x0 + x1)) : 0.f;
  const float fcy = (y0 <= y1) ? static_cast<float>(0.5 * (y0 + y1)) : 0.f;
  const double cx = fcx, cy = fcy;
  const CsrView val{vvx, vvy};
  // Voronoi frame: the centroid rounded to f32, so p0' = p0 - c is below half
  // an ulp of |p0| (< 6e-8 max(1, |p0|), far inside the 1e-5 band) and is
  // taken as 0 -- the block carries the n generators only
  float gcx = fcx, gcy = fcy;
  if (status == 0 && (a.kinds & kKindVoronoi)) {
    double px, py;
    centroid_exact(val, n, &px, &py);
    a.inner[i] = make_double2(px, py);
    gcx = static_cast<float>(px);
    gcy = static_cast<float>(py);
    for (int k = 0; k < n && status == 0; ++k) {
      double2 g;
      status = reflect_exact(val(k), val((k + 1) % n), px, py, &g);
      if (status) break;
      a.outer[s + k] = g;
      a.gen[blk + 2 + k] = local(g, gcx, gcy);
    }
  }
  // offset / crossing: v_{n-1}, v_0 .. v_{n-1} -- the leading copy of the last
  // vertex closes the ring without a register pair held across the row loop
  // (that pair costs the crossing kernel a CTA per SM or a spill)
  if (status == 0 && (a.kinds & kKindOffset) && n > 0) {
    a.ccw[blk + 2] = local(val(n - 1), cx, cy);
    for (int k = 0; k < n; ++k) a.ccw[blk + 3 + k] = local(val(k), cx, cy);
  }
  if ((a.kinds & kKindCrossing) && n > 0) {
    a.raw[blk + 2] = local(raw(n - 1), cx, cy);
    for (int k = 0; k < n; ++k) a.raw[blk + 3 + k] = local(raw(k), cx, cy);
  }
  a.status[i] = status;
  // a failed polygon tests outside under Voronoi / sign-of-offset (crossing
  // ignores the flag: it accepts any polygon)
  const bool bad = convex && status != 0;
  const float nbits = __uint_as_float(static_cast<uint32_t>(n) | (bad ? kRangeInvalid : 0u));
  for (float2* t : {a.gen, a.ccw, a.raw}) t[blk] = make_float2(nbits, 0.f);
  // the raw rows equal the validated ones unless validation reversed or
  // rejected the polygon (or did not run)
  if (!convex || bad || rev)
    a.raw[blk] = make_float2(__uint_as_float(__float_as_uint(nbits) | kRawDiffers), 0.f);
  a.gen[blk + 1] = make_float2(gcx, gcy);
  a.ccw[blk + 1] = make_float2(fcx, fcy);
  a.raw[blk + 1] = make_float2(fcx, fcy);
}

#ifndef VPIPG_GP
#define VPIPG_GP 1
#endif
#ifndef VPIPG_GMINB
#define VPIPG_GMINB 8
#endif
constexpr int kGP = VPIPG_GP;  // pairs per lane
#ifndef VPIPG_GMINB_ALL
#define VPIPG_GMINB_ALL 5  // the fused join keeps two walks' state live: 48 registers (6 CTAs: 7.75 ms, 5: 6.98, 4: 7.27 at C4)
#endif
constexpr int kGThreads = 256;

// 32-byte (256-bit) read-only load: four rows (or the header + two rows).
struct Rows4 {
  float v[8];
};
__device__ __forceinline__ Rows4 ld256(const float2* p) {
  Rows4 r;
  asm volatile("ld.global.nc.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=f"(r.v[0]), "=f"(r.v[1]), "=f"(r.v[2]), "=f"(r.v[3]), "=f"(r.v[4]),
                 "=f"(r.v[5]), "=f"(r.v[6]), "=f"(r.v[7])
               : "l"(p));
  return r;
}

// Per-engine accumulation over a polygon's rows (row 0 first): Voronoi rows
// are the n outer generators (the inner one is the origin); offset / crossing
// rows are v_{n-1}, v_0 .. v_{n-1}, row 0 only seeding the previous vertex.
template <int kEngine>
struct RowAcc {
  uint32_t acc = 0;
  float pa = 0.f, pb = 0.f;  // previous row relative to q' (offset / crossing), or |q'-p0'|^2
  __device__ __forceinline__ void first(float qx, float qy, float rx, float ry) {
    if (kEngine == 0) {
      pa = fmaf(qx, qx, qy * qy);  // inner_sq with p0' = 0
      next(qx, qy, rx, ry);
    } else {
      pa = qx - rx;
      pb = qy - ry;
    }
  }
  __device__ __forceinline__ void next(float qx, float qy, float rx, float ry) {
    const float a = qx - rx, b = qy - ry;
    if (kEngine == 0) {  // |q'-pk'|^2 - |q'-p0'|^2 >= 0 for every outer generator
      acc |= __float_as_uint(fmaf(a, a, b * b) - pa);
    } else {
      const float s = fmaf(pa, b, -(a * pb));  // (q - v_j) x (q - v_i)
      if (kEngine == 1) {
        acc |= __float_as_uint(s);
      } else {
        const uint32_t hi = __float_as_uint(b), hj = __float_as_uint(pb);
        acc ^= (hi ^ hj) & (__float_as_uint(s) ^ hi);
      }
      pa = a;
      pb = b;
    }
  }
  __device__ __forceinline__ bool inside() const {
    return kEngine == 2 ? (acc >> 31) != 0 : !(acc >> 31);
  }
};

template <int kEngine>  // 0 voronoi, 1 offset, 2 crossing
__global__ void __launch_bounds__(kGThreads, VPIPG_GMINB) gather_kernel(const DbTables t,
                                                                        const GatherArgs a) {
  const int lane = threadIdx.x & 31;
  const uint64_t gwarp = (uint64_t)blockIdx.x * (kGThreads / 32) + (threadIdx.x >> 5);
  const uint64_t stride = (uint64_t)gridDim.x * (kGThreads / 32) * 32 * kGP;
  const float2* tab = kEngine == 0 ? t.gen : kEngine == 1 ? t.ccw : t.raw;
  uint32_t count = 0;
  for (uint64_t base = gwarp * 32 * kGP; base < a.m; base += stride) {
    float qx[kGP], qy[kGP];
    const float2* blk[kGP];
    uint32_t rows[kGP];  // rows to read (n Voronoi, n + 1 otherwise), 0 = outside regardless
    bool ok[kGP];
    RowAcc<kEngine> r[kGP];
    uint32_t rmax = 0;
#pragma unroll
    for (int p = 0; p < kGP; ++p) {
      const uint64_t j = base + 32u * p + lane;
      ok[p] = j < a.m;
      const uint32_t id = ok[p] ? __ldcs(a.ids + j) : 0u;
      const float x = ok[p] ? __ldcs(a.xs + j) : 0.f;
      const float y = ok[p] ? __ldcs(a.ys + j) : 0.f;
      ok[p] = ok[p] && id < t.npoly;
      blk[p] = tab + (uint64_t)(ok[p] ? id : 0u) * t.stride;
      const Rows4 h = ok[p] ? ld256(blk[p]) : Rows4{};
      const uint32_t nf = __float_as_uint(h.v[0]);
      // a polygon that failed validation only disables the convex engines: ray
      // crossing takes the raw vertices of any polygon (vpip.cpp:120-128)
      if (kEngine != 2) ok[p] = ok[p] && !(nf & kRangeInvalid);
      const uint32_t n = nf & ~(kRangeInvalid | kRawDiffers);
      rows[p] = (ok[p] && n > 0) ? (kEngine == 0 ? n : n + 1) : 0u;
      qx[p] = x - h.v[2];  // exact for points near their polygon (Sterbenz)
      qy[p] = y - h.v[3];
      if (rows[p] > 0) r[p].first(qx[p], qy[p], h.v[4], h.v[5]);
      if (rows[p] > 1) r[p].next(qx[p], qy[p], h.v[6], h.v[7]);
      rmax = rows[p] > rmax ? rows[p] : rmax;
    }
    if (kEngine == 1) {
      // sign-of-offset: per-row predicates (the split loop below spills its
      // extra live values at 32 registers for this engine)
      for (uint32_t k = 2; k < rmax; k += 4) {  // rows k .. k+3 = slots k+2 .. k+5
#pragma unroll
        for (int p = 0; p < kGP; ++p) {
          if (k < rows[p]) {
            const Rows4 q4 = ld256(blk[p] + k + 2);
#pragma unroll
            for (int u = 0; u < 4; ++u)
              if (k + u < rows[p]) r[p].next(qx[p], qy[p], q4.v[2 * u], q4.v[2 * u + 1]);
          }
        }
      }
    } else {
#pragma unroll
      for (int p = 0; p < kGP; ++p) {
        // full 4-row chunks without per-row predicates, then a tail of <= 3
        uint32_t k = 2;
        for (; k + 3 < rows[p]; k += 4) {
          const Rows4 q4 = ld256(blk[p] + k + 2);
#pragma unroll
          for (int u = 0; u < 4; ++u) r[p].next(qx[p], qy[p], q4.v[2 * u], q4.v[2 * u + 1]);
        }
        if (k < rows[p]) {
          const Rows4 q4 = ld256(blk[p] + k + 2);
          r[p].next(qx[p], qy[p], q4.v[0], q4.v[1]);
          if (k + 1 < rows[p]) r[p].next(qx[p], qy[p], q4.v[2], q4.v[3]);
          if (k + 2 < rows[p]) r[p].next(qx[p], qy[p], q4.v[4], q4.v[5]);
        }
      }
    }
    bool in[kGP];
#pragma unroll
    for (int p = 0; p < kGP; ++p) {
      in[p] = ok[p] && rows[p] > 0 && r[p].inside();
      // a NaN coordinate: the reference's IEEE answer (Voronoi compares are
      // false -> outside; sign-of-offset raises no flag -> inside)
      if (kEngine != 2 && ok[p] && rows[p] > 0 && (qx[p] != qx[p] || qy[p] != qy[p]))
        in[p] = kEngine == 1;
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

// Walk rows 2 .. rows-1 of a block (rows 0 and 1 came with the header load)
// into one accumulator, or into two that share every row (kBoth: offset +
// crossing over the same vertex rows).
template <bool kBoth, class R1, class R2>
__device__ __forceinline__ void walk(const float2* blk, uint32_t rows, float qx, float qy, R1& r1,
                                     R2& r2) {
  uint32_t k = 2;
  for (; k + 3 < rows; k += 4) {
    const Rows4 q4 = ld256(blk + k + 2);
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      r1.next(qx, qy, q4.v[2 * u], q4.v[2 * u + 1]);
      if (kBoth) r2.next(qx, qy, q4.v[2 * u], q4.v[2 * u + 1]);
    }
  }
  if (k < rows) {
    const Rows4 q4 = ld256(blk + k + 2);
#pragma unroll
    for (int u = 0; u < 3; ++u)
      if (k + u < rows) {
        r1.next(qx, qy, q4.v[2 * u], q4.v[2 * u + 1]);
        if (kBoth) r2.next(qx, qy, q4.v[2 * u], q4.v[2 * u + 1]);
      }
  }
}

// Fused join: every (point, id) pair is read once and tested by all three
// engines. Voronoi walks the generator block; sign-of-offset and crossing
// share ONE walk over the raw vertex rows (the same rows and frame as the
// validated ones unless the header says kRawDiffers, when offset walks its own
// block), so a pair touches two polygon blocks instead of three.
__global__ void __launch_bounds__(kGThreads, VPIPG_GMINB_ALL)
    gather_all_kernel(const DbTables t, const GatherArgs av, const GatherArgs ao,
                      const GatherArgs ac) {
  const int lane = threadIdx.x & 31;
  const uint64_t gwarp = (uint64_t)blockIdx.x * (kGThreads / 32) + (threadIdx.x >> 5);
  const uint64_t stride = (uint64_t)gridDim.x * (kGThreads / 32) * 32;
  uint32_t cnt[3] = {0, 0, 0};
  for (uint64_t base = gwarp * 32; base < av.m; base += stride) {
    const uint64_t j = base + lane;
    bool ok = j < av.m;
    const uint32_t id = ok ? __ldcs(av.ids + j) : 0u;
    const float x = ok ? __ldcs(av.xs + j) : 0.f;
    const float y = ok ? __ldcs(av.ys + j) : 0.f;
    ok = ok && id < t.npoly;
    const uint64_t off = (uint64_t)(ok ? id : 0u) * t.stride;
    bool in[3] = {false, false, false};
    // ---- Voronoi: generator block, its own frame ----
    {
      const float2* blk = t.gen + off;
      const Rows4 h = ok ? ld256(blk) : Rows4{};
      const uint32_t nf = __float_as_uint(h.v[0]);
      const uint32_t n = nf & ~(kRangeInvalid | kRawDiffers);
      const uint32_t rows = (ok && !(nf & kRangeInvalid)) ? n : 0u;
      const float qx = x - h.v[2], qy = y - h.v[3];
      RowAcc<0> r;
      if (rows > 0) r.first(qx, qy, h.v[4], h.v[5]);
      if (rows > 1) r.next(qx, qy, h.v[6], h.v[7]);
      walk<false>(blk, rows, qx, qy, r, r);
      in[0] = rows > 0 && (qx != qx || qy != qy ? false : r.inside());
    }
    // ---- crossing (+ offset when the rows coincide): raw block ----
    {
      const float2* blk = t.raw + off;
      const Rows4 h = ok ? ld256(blk) : Rows4{};
      const uint32_t nf = __float_as_uint(h.v[0]);
      const uint32_t n = nf & ~(kRangeInvalid | kRawDiffers);
      const uint32_t rows = (ok && n > 0) ? n + 1 : 0u;
      const bool shared = !(nf & kRawDiffers);
      const float qx = x - h.v[2], qy = y - h.v[3];
      RowAcc<2> rc;
      RowAcc<1> ro;
      if (rows > 0) {
        rc.first(qx, qy, h.v[4], h.v[5]);
        ro.first(qx, qy, h.v[4], h.v[5]);
      }
      if (rows > 1) {
        rc.next(qx, qy, h.v[6], h.v[7]);
        ro.next(qx, qy, h.v[6], h.v[7]);
      }
      if (shared)
        walk<true>(blk, rows, qx, qy, rc, ro);
      else
        walk<false>(blk, rows, qx, qy, rc, rc);
      in[2] = rows > 0 && rc.inside();
      const bool nan = qx != qx || qy != qy;
      if (shared) {
        in[1] = rows > 0 && (nan || ro.inside());
      } else if (ok && !(nf & kRangeInvalid)) {
        // reversed by validation: offset walks the validated (CCW) rows
        const float2* cb = t.ccw + off;
        const Rows4 hc = ld256(cb);
        const float cx = x - hc.v[2], cy = y - hc.v[3];
        RowAcc<1> r;
        r.first(cx, cy, hc.v[4], hc.v[5]);
        if (rows > 1) r.next(cx, cy, hc.v[6], hc.v[7]);
        walk<false>(cb, rows, cx, cy, r, r);
        in[1] = rows > 0 && (nan || r.inside());
      }
    }
    const GatherArgs* args[3] = {&av, &ao, &ac};
#pragma unroll
    for (int e = 0; e < 3; ++e) {
      const GatherArgs& a = *args[e];
      const uint32_t w = __ballot_sync(0xffffffffu, in[e]);
      cnt[e] += in[e];
      if (a.words && lane == 0) a.words[base >> 5] = w;
      if (a.bytes && j < a.m) a.bytes[j] = in[e] ? 1 : 0;
    }
  }
  const GatherArgs* args[3] = {&av, &ao, &ac};
#pragma unroll
  for (int e = 0; e < 3; ++e) {
    uint32_t c = cnt[e];
#pragma unroll
    for (int s = 16; s > 0; s >>= 1) c += __shfl_xor_sync(0xffffffffu, c, s);
    if (lane == 0 && args[e]->inside && c) atomicAdd(args[e]->inside, (unsigned long long)c);
  }
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

cudaError_t launch_gather_all(const DbTables& t, const GatherArgs* a, cudaStream_t stream) {
  if (a[0].m == 0) return cudaSuccess;
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const uint64_t warps = (a[0].m + 31) / 32;
  const uint64_t blocks = (warps + kGThreads / 32 - 1) / (kGThreads / 32);
  const uint64_t cap = (uint64_t)sms * VPIPG_GMINB_ALL;
  const int grid = static_cast<int>(blocks < cap ? blocks : cap);
  gather_all_kernel<<<grid, kGThreads, 0, stream>>>(t, a[0], a[1], a[2]);
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
