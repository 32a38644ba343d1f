// csr.cu -- polygon-database join (BASELINE config 4): batched device
// preparation of a CSR polygon table and the gather test kernels.
//
// prep_csr_kernel, one thread per polygon:
//   validate_polygon (geometry.cpp:53-98) -> per-polygon status and
//   orientation, to_voronoi (voronoi.cpp:60-71) with the reference's exact f64
//   arithmetic (the generator set vpipg_db_generators reads back), then ONE
//   32-byte-aligned record per polygon (vpipg_internal.h): a 32-byte header
//   (n and flags, frame origin c, the centroid p0' - the inner generator - and
//   the closing vertex) and the raw vertex rows, f32 in the polygon-local
//   frame (c = the f32 bounding-box centre). Records are packed back to back
//   (per-polygon offsets), so one polygon with many vertices costs only its
//   own rows.
// gather_all_kernel / gather_kernel: every (point, polygon id) pair reads its
//   polygon's header and walks its rows once, in 32-byte loads, from the
//   L2-resident records; q' = q - c is exact in f32 (Sterbenz) for points near
//   their polygon. For the edge v_j -> v_i of consecutive rows:
//     Voronoi    outer generator g = p0' - f n (the mirror of the centroid
//                across the edge line with normal n, reflect_generator's Eq. 8;
//                prep stores the scalar f per edge, n comes from the two rows),
//                inside iff |q'-g|^2 >= |q'-p0'|^2 for every edge
//                (engines.cpp:85-98, ties inside)
//     offset     s = (q - v_j) x (q - v_i) >= 0 in the validated (CCW) order,
//                i.e. s <= 0 on raw rows that validation reversed
//                (engines.cpp:150-152)
//     crossing   in_range = H_i ^ H_j, on_left = sign(s) ^ H_i (H = [v.y > qy]),
//                parity by XOR (engines.cpp:187-196), on the raw order
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
  float2* r = a.recs + 4 * (uint64_t)a.rec[i];
  const CsrView raw{a.vx + s, a.vy + s};
  int status = 0;
  bool rev = false;
  const bool convex = a.kinds & (kKindVoronoi | kKindOffset);
  if (convex) status = validate_exact(raw, n, &rev);
  double x0 = INFINITY, x1 = -INFINITY, y0 = INFINITY, y1 = -INFINITY;
  for (int k = 0; k < n; ++k) {
    const double2 p = raw(k);
    if (isfinite(p.x) && isfinite(p.y)) {
      x0 = fmin(x0, p.x); x1 = fmax(x1, p.x);
      y0 = fmin(y0, p.y); y1 = fmax(y1, p.y);
    }
  }
  // polygon-local frame: f32 centre of the bounding box
  const float fcx = (x0 <= x1) ? static_cast<float>(0.5 * (x0 + x1)) : 0.f;
  const float fcy = (y0 <= y1) ? static_cast<float>(0.5 * (y0 + y1)) : 0.f;
  const double cx = fcx, cy = fcy;
  // validated (CCW) order = the raw rows read backwards when reversed
  auto val = [&](int k) { return raw(rev ? n - 1 - k : k); };
  float2 p0 = make_float2(0.f, 0.f);
  // record body: groups of 8 edges, group g at slot 4 + 12 g: its 8 rows, then
  // its 8 f values (vpipg_internal.h)
  auto row = [&](int k) -> float2& { return r[4 + 12 * (k >> 3) + (k & 7)]; };
  auto fval = [&](int k) -> float& {
    return reinterpret_cast<float*>(r + 12 + 12 * (k >> 3))[k & 7];
  };
  if (status == 0 && (a.kinds & kKindVoronoi)) {
    double px, py;
    centroid_exact(val, n, &px, &py);
    a.inner[i] = make_double2(px, py);
    p0 = local(make_double2(px, py), cx, cy);
    for (int k = 0; k < n && status == 0; ++k) {
      double2 g;
      status = reflect_exact(val(k), val((k + 1) % n), px, py, &g);
      if (status == 0) a.outer[s + k] = g;
    }
    // the outer generator of raw edge v_{k-1} -> v_k as g = p0 - f_k n_k with
    // n_k = (v_{k-1}.y - v_k.y, v_k.x - v_{k-1}.x) from the f32 rows the
    // kernels read: f_k = -(g - p0).n_k / |n_k|^2 (g - p0 is parallel to n_k;
    // the rows' rounding only turns it by < 1e-7 rad)
    for (int k = 0; k < n && status == 0; ++k) {
      const float2 vj = local(raw((k + n - 1) % n), cx, cy), vi = local(raw(k), cx, cy);
      const double nx = static_cast<double>(vj.y) - vi.y, ny = static_cast<double>(vi.x) - vj.x;
      const int vk = rev ? n - 1 - k : (k + n - 1) % n;  // the validated edge this raw edge is
      const double2 g = a.outer[s + vk];
      const double dd = nx * nx + ny * ny;
      fval(k) = dd > 0.0 ? static_cast<float>(-((g.x - px) * nx + (g.y - py) * ny) / dd) : 0.f;
    }
  }
  a.status[i] = status;
  // a failed polygon tests outside under Voronoi / sign-of-offset (crossing
  // ignores the flag: it accepts any polygon)
  const uint32_t nf = static_cast<uint32_t>(n) | ((convex && status != 0) ? kRangeInvalid : 0u) |
                      (rev ? kReversed : 0u);
  r[0] = make_float2(__uint_as_float(nf), 0.f);
  r[1] = make_float2(fcx, fcy);
  r[2] = p0;
  if (n > 0) {
    r[3] = local(raw(n - 1), cx, cy);
    for (int k = 0; k < n; ++k) row(k) = local(raw(k), cx, cy);
  }
}

#ifndef VPIPG_GMINB
#define VPIPG_GMINB 5
#endif
#ifndef VPIPG_GSTREAM_AHEAD
#define VPIPG_GSTREAM_AHEAD 1
#endif
#ifndef VPIPG_GMINB_ALL
#define VPIPG_GMINB_ALL 4
#endif
constexpr int kGThreads = 256;

// 32-byte (256-bit) read-only load: four rows (or the header).
struct Rows4 {
  float v[8];
};
__device__ __forceinline__ Rows4 ld256(const float2* p) {
  Rows4 r;
  // not volatile: the compiler may hoist the next chunk's load above this
  // chunk's arithmetic (the tables are read-only for the kernel's lifetime)
  asm("ld.global.nc.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=f"(r.v[0]), "=f"(r.v[1]), "=f"(r.v[2]), "=f"(r.v[3]), "=f"(r.v[4]),
                 "=f"(r.v[5]), "=f"(r.v[6]), "=f"(r.v[7])
               : "l"(p));
  return r;
}


// The three engines' state for one pair over one polygon's edges.
template <bool kV, bool kO, bool kC>
struct PairAcc {
  float qx, qy;       // q' (local frame)
  float qpx, qpy;     // q' - p0' (p0' the inner generator)
  float d0;           // |q' - p0'|^2
  float pa, pb;       // q' - v_j of the previous row
  float px, py;       // v_j' itself (the Voronoi edge normal)
  uint32_t vor = 0;   // sign bits of |q'-g|^2 - |q'-p0'|^2 (any set: outside)
  uint32_t off = 0;   // sign bits of the oriented cross products (any set: outside)
  uint32_t par = 0;   // crossing parity (bit 31)
  uint32_t flip = 0;  // 0x80000000 when the raw rows run clockwise

  __device__ __forceinline__ void start(float x, float y, float cx, float cy, float gx, float gy,
                                        float lx, float ly, uint32_t rev) {
    qx = x - cx;  // exact for points near their polygon (Sterbenz)
    qy = y - cy;
    if (kV) {
      qpx = qx - gx;
      qpy = qy - gy;
      d0 = fmaf(qpx, qpx, qpy * qpy);
    }
    pa = qx - lx;
    pb = qy - ly;
    px = lx;
    py = ly;
    flip = rev ? 0x80000000u : 0u;
  }
  // edge v_j -> v_i with v_j the previous row, v_i = (rx, ry) and f the
  // edge's generator coefficient (the outer generator g = p0' - f n)
  __device__ __forceinline__ void edge(float rx, float ry, float f) {
    const float a = qx - rx, b = qy - ry;
    if (kV) {
      // n = (v_j.y - v_i.y, v_i.x - v_j.x), the edge line's normal
      // (edge_coefficients, voronoi.cpp:23-31); q' - g = (q' - p0') + f n
      const float nx = py - ry, ny = rx - px;
      const float ex = fmaf(f, nx, qpx), ey = fmaf(f, ny, qpy);
      vor |= __float_as_uint(fmaf(ex, ex, ey * ey) - d0);  // |q'-g|^2 - |q'-p0'|^2
    }
    if (kO || kC) {
      const float s = fmaf(pa, b, -(a * pb));  // (q - v_j) x (q - v_i)
      if (kO) off |= __float_as_uint(s) ^ flip;
      if (kC) {
        const uint32_t hi = __float_as_uint(b), hj = __float_as_uint(pb);
        par ^= (hi ^ hj) & (__float_as_uint(s) ^ hi);
      }
    }
    pa = a;
    pb = b;
    px = rx;
    py = ry;
  }
};

// One pair against its polygon's record; `in` receives the requested engines'
// answers (a NaN coordinate gets the reference's IEEE answer: Voronoi outside,
// sign-of-offset inside).
template <bool kV, bool kO, bool kC>
__device__ __forceinline__ void test_pair(const DbTables& t, bool ok, uint32_t id, float x, float y,
                                          bool (&in)[3]) {
  // fixed-stride records (t.stride 32-byte units, id * stride) when the sizes
  // are uniform enough; per-polygon offsets otherwise (one dependent load more)
  const uint64_t unit = t.stride ? (uint64_t)id * t.stride : (uint64_t)(ok ? __ldg(t.rec + id) : 0u);
  const float2* r = t.recs + 4 * (ok ? unit : 0u);
  const Rows4 h = ld256(r);
  const uint32_t nf = __float_as_uint(h.v[0]);
  const uint32_t n = ok ? nf & kNMask : 0u;
  PairAcc<kV, kO, kC> acc;
  acc.start(x, y, h.v[2], h.v[3], h.v[4], h.v[5], h.v[6], h.v[7], nf & kReversed);
  // group 0 (edges 0..7) is read together with the header -- its address does
  // not depend on n -- and later groups after it, three 32-byte loads each
  auto group = [&](uint32_t g, const Rows4& h0, const Rows4& h1, const Rows4& f) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      if (8 * g + u < n) {
        const Rows4& q = u < 4 ? h0 : h1;
        acc.edge(q.v[2 * (u & 3)], q.v[2 * (u & 3) + 1], kV ? f.v[u] : 0.f);
      }
    }
  };
  {
    const Rows4 r0 = ld256(r + 4), r1 = ld256(r + 8);
    const Rows4 f0 = kV ? ld256(r + 12) : Rows4{};
    group(0, r0, r1, f0);
  }
  for (uint32_t g = 1; 8 * g < n; ++g) {
    const float2* b = r + 4 + 12 * g;
    // the second row chunk only when the group has more than 4 edges
    const Rows4 r0 = ld256(b), r1 = 8 * g + 4 < n ? ld256(b + 4) : Rows4{};
    const Rows4 f0 = kV ? ld256(b + 8) : Rows4{};
    group(g, r0, r1, f0);
  }
  const bool convex_ok = n > 0 && !(nf & kRangeInvalid);
  const bool nan = acc.qx != acc.qx || acc.qy != acc.qy;
  in[0] = kV && convex_ok && !nan && !(acc.vor >> 31);
  in[1] = kO && convex_ok && (nan || !(acc.off >> 31));
  in[2] = kC && n > 0 && (acc.par >> 31);
}

// kMask: bit e = engine e (Voronoi, offset, crossing) of this launch; a[e]
// its outputs (all share xs, ys, ids, m)
template <int kMask>
__global__ void __launch_bounds__(kGThreads, kMask == 7 ? VPIPG_GMINB_ALL : VPIPG_GMINB)
    gather_kernel(const DbTables t, const GatherArgs av, const GatherArgs ao, const GatherArgs ac) {
  constexpr bool kV = kMask & 1, kO = kMask & 2, kC = kMask & 4;
  const GatherArgs& a0 = kV ? av : kO ? ao : ac;
  const int lane = threadIdx.x & 31;
  const uint64_t gwarp = (uint64_t)blockIdx.x * (kGThreads / 32) + (threadIdx.x >> 5);
  const uint64_t stride = (uint64_t)gridDim.x * (kGThreads / 32) * 32;
  uint32_t cnt[3] = {0, 0, 0};
  // the next pair's stream words are loaded one iteration ahead
  auto load = [&](uint64_t j, uint32_t& id, float& x, float& y) {
    const bool in = j < a0.m;
    id = in ? __ldcs(a0.ids + j) : 0u;
    x = in ? __ldcs(a0.xs + j) : 0.f;
    y = in ? __ldcs(a0.ys + j) : 0.f;
  };
  uint32_t nid;
  float nx, ny;
  load(gwarp * 32 + lane, nid, nx, ny);
  for (uint64_t base = gwarp * 32; base < a0.m; base += stride) {
    const uint64_t j = base + lane;
    const uint32_t id = nid;
    const float x = nx, y = ny;
    if (VPIPG_GSTREAM_AHEAD) load(j + stride, nid, nx, ny);
    bool ok = j < a0.m;
    ok = ok && id < t.npoly;
    bool in[3];
    test_pair<kV, kO, kC>(t, ok, id, x, y, in);
    if (!VPIPG_GSTREAM_AHEAD) load(j + stride, nid, nx, ny);
    const GatherArgs* args[3] = {&av, &ao, &ac};
#pragma unroll
    for (int e = 0; e < 3; ++e) {
      if (!(kMask & (1 << e))) continue;
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
    if (!(kMask & (1 << e))) continue;
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

namespace {
template <int kMask>
cudaError_t launch_gather_mask(const DbTables& t, const GatherArgs& av, const GatherArgs& ao,
                               const GatherArgs& ac, uint64_t m, cudaStream_t stream) {
  int sms = 0, per_sm = 0;
  auto k = gather_kernel<kMask>;
  const cudaError_t e = launch_config(reinterpret_cast<const void*>(k), kGThreads, 0, &sms, &per_sm);
  if (e != cudaSuccess) return e;
  const uint64_t warps = (m + 31) / 32;
  const uint64_t blocks = (warps + kGThreads / 32 - 1) / (kGThreads / 32);
  const uint64_t cap = (uint64_t)sms * per_sm;
  k<<<static_cast<int>(blocks < cap ? blocks : cap), kGThreads, 0, stream>>>(t, av, ao, ac);
  return cudaGetLastError();
}
}  // namespace

cudaError_t launch_gather(const DbTables& t, int engine, const GatherArgs& a, cudaStream_t stream) {
  if (a.m == 0) return cudaSuccess;
  switch (engine) {
    case 0: return launch_gather_mask<1>(t, a, a, a, a.m, stream);
    case 1: return launch_gather_mask<2>(t, a, a, a, a.m, stream);
    default: return launch_gather_mask<4>(t, a, a, a, a.m, stream);
  }
}

cudaError_t launch_gather_all(const DbTables& t, const GatherArgs* a, cudaStream_t stream) {
  if (a[0].m == 0) return cudaSuccess;
  return launch_gather_mask<7>(t, a[0], a[1], a[2], a[0].m, stream);
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
