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
//                f and n formed in registers from the two rows and p0'),
//                inside iff |q'-g|^2 >= |q'-p0'|^2 for every edge
//                (engines.cpp:85-98, ties inside)
//     offset     s = (q - v_j) x (q - v_i) >= 0 in the validated (CCW) order
//                (engines.cpp:150-152)
//     crossing   in_range = H_i ^ H_j, on_left = sign(s) ^ H_i (H = [v.y > qy]),
//                parity by XOR (engines.cpp:187-196); the rows are stored in
//                the validated order, the reverse of a clockwise raw polygon,
//                which leaves the crossing parity unchanged
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
    // the rows in the validated order (the crossing parity does not depend
    // on the direction of travel), padded to whole 4-row chunks with copies
    // of the last row: a repeated row is an empty edge every engine ignores
    const float2 last = local(val(n - 1), cx, cy);
    r[3] = last;
    for (int k = 0; k < n; ++k) r[4 + k] = local(val(k), cx, cy);
    for (int k = n; k < 4 * ((n + 3) / 4); ++k) r[4 + k] = last;
  }
}

#ifndef VPIPG_GMINB
#define VPIPG_GMINB 5
#endif
#ifndef VPIPG_GSTREAM_AHEAD
#define VPIPG_GSTREAM_AHEAD 1
#endif
#ifndef VPIPG_GMINB_ALL
#define VPIPG_GMINB_ALL 5
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


// MUFU.RCP (about 1 ulp): the generator it places is off by ~1e-7 of the
// polygon's extent, far inside the band
__device__ __forceinline__ float rcp_approx(float x) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

// three-input minimum (FMNMX3; NaN operands are ignored)
__device__ __forceinline__ float min3(float a, float b, float c) {
  float r;
  asm("min.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
  return r;
}

// The three engines' state for one pair over one polygon's edges.
template <bool kV, bool kO, bool kC>
struct PairAcc {
  float qx, qy;       // q' (local frame)
  float qpx, qpy;     // 2 (q' - p0') (p0' the inner generator)
  float tgx, tgy;     // 2 p0'
  float pa, pb;       // q' - v_j of the previous row
  float px, py;       // v_j' itself
  // running minima of |q'-g|^2 - |q'-p0'|^2 and of the cross products over
  // the edges so far (negative: outside), two edges per three-input min (it
  // issues like one LOP3 per two edges instead of one per edge)
  float vor = INFINITY, off = INFINITY;
  uint32_t par = 0;   // crossing parity (bit 31)

  __device__ __forceinline__ void start(float x, float y, float cx, float cy, float gx, float gy,
                                        float lx, float ly) {
    qx = x - cx;  // exact for points near their polygon (Sterbenz)
    qy = y - cy;
    if (kV) {
      qpx = 2.f * (qx - gx);
      qpy = 2.f * (qy - gy);
      tgx = gx + gx;
      tgy = gy + gy;
    }
    pa = qx - lx;
    pb = qy - ly;
    px = lx;
    py = ly;
  }
  // edge v_j -> v_i, v_j the previous row and v_i = (rx, ry), in the validated
  // (counter-clockwise) order. A repeated row (the chunk padding) is an empty
  // edge: n = 0 gives f = 0 and g = p0', s = +0, no crossing.
  __device__ __forceinline__ void edge(float rx, float ry, float& dv, float& s) {
    const float a = qx - rx, b = qy - ry;
    dv = INFINITY;
    s = 0.f;
    if (kV) {
      // the outer generator g = p0' - f n, the mirror of p0' across the edge
      // line (reflect_generator, voronoi.cpp:46-58) with n = (v_j.y - v_i.y,
      // v_i.x - v_j.x) (edge_coefficients, voronoi.cpp:23-31) and
      // f = 2 (p0' - v_j).n / |n|^2, formed in registers from the two rows
      const float nx = py - ry, ny = rx - px;
      const float dx = fmaf(-2.f, px, tgx), dy = fmaf(-2.f, py, tgy);  // 2 (p0' - v_j)
      const float nn = fmaf(nx, nx, fmaf(ny, ny, 1e-30f));
      const float f = fmaf(dx, nx, dy * ny) * rcp_approx(nn);
      // |q'-g|^2 - |q'-p0'|^2 = |(q'-p0') + f n|^2 - |q'-p0'|^2
      //                      = f (f |n|^2 + 2 (q'-p0').n), expanded (no cancellation)
      dv = f * fmaf(f, nn, fmaf(qpx, nx, qpy * ny));
    }
    if (kO || kC) {
      // (q - v_j) x (q - v_i), exactly +0 for v_i = v_j (no contraction)
      s = __fsub_rn(__fmul_rn(pa, b), __fmul_rn(a, pb));
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
  __device__ __forceinline__ void chunk(const Rows4& c) {
#pragma unroll
    for (int u = 0; u < 4; u += 2) {
      float v0, s0, v1, s1;
      edge(c.v[2 * u], c.v[2 * u + 1], v0, s0);
      edge(c.v[2 * u + 2], c.v[2 * u + 3], v1, s1);
      if (kV) vor = min3(vor, v0, v1);
      if (kO) off = min3(off, s0, s1);
    }
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
  // the header and the first two 4-row chunks in one round trip (their
  // addresses do not depend on n; every record holds at least two chunks),
  // later chunks two at a time once n is known
  const Rows4 h = ld256(r), c0 = ld256(r + 4), c1 = ld256(r + 8);
  const uint32_t nf = __float_as_uint(h.v[0]);
  const uint32_t n = ok ? nf & kNMask : 0u;
  PairAcc<kV, kO, kC> acc;
  acc.start(x, y, h.v[2], h.v[3], h.v[4], h.v[5], h.v[6], h.v[7]);
  acc.chunk(c0);
  if (n > 4) acc.chunk(c1);
  for (uint32_t c = 2; 4 * c < n; c += 2) {
    const Rows4 ca = ld256(r + 4 + 4 * c);
    const bool two = 4 * c + 4 < n;
    const Rows4 cb = two ? ld256(r + 8 + 4 * c) : Rows4{};
    acc.chunk(ca);
    if (two) acc.chunk(cb);
  }
  const bool convex_ok = n > 0 && !(nf & kRangeInvalid);
  const bool nan = acc.qx != acc.qx || acc.qy != acc.qy;
  in[0] = kV && convex_ok && !nan && !(acc.vor < 0.f);
  in[1] = kO && convex_ok && (nan || !(acc.off < 0.f));
  in[2] = kC && n > 0 && (acc.par >> 31);
}

// kMask: bit e = engine e (Voronoi, offset, crossing) of this launch; a[e]
// its outputs (all share xs, ys, ids, m). kBytes: some engine wants a byte
// mask (decided per launch, so the common words-only launch carries no byte
// stores or their address arithmetic).
template <int kMask, bool kBytes>
__global__ void __launch_bounds__(kGThreads, kMask == 7 ? VPIPG_GMINB_ALL : VPIPG_GMINB)
    gather_kernel(const DbTables t, const GatherArgs av, const GatherArgs ao, const GatherArgs ac) {
  constexpr bool kV = kMask & 1, kO = kMask & 2, kC = kMask & 4;
  const GatherArgs& a0 = kV ? av : kO ? ao : ac;
  const int lane = threadIdx.x & 31;
  const uint64_t gwarp = (uint64_t)blockIdx.x * (kGThreads / 32) + (threadIdx.x >> 5);
  const uint64_t stride = (uint64_t)gridDim.x * (kGThreads / 32) * 32;
  // warp-wide inside counts: every lane adds the popcount of the (uniform)
  // ballot word, lane 0 flushes
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
      cnt[e] += __popc(w);
      if (a.words && lane == 0) a.words[base >> 5] = w;
      if (kBytes && a.bytes && j < a.m) a.bytes[j] = in[e] ? 1 : 0;
    }
  }
  const GatherArgs* args[3] = {&av, &ao, &ac};
#pragma unroll
  for (int e = 0; e < 3; ++e) {
    if (!(kMask & (1 << e))) continue;
    if (lane == 0 && args[e]->inside && cnt[e]) atomicAdd(args[e]->inside, (unsigned long long)cnt[e]);
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
  const bool bytes = ((kMask & 1) && av.bytes) || ((kMask & 2) && ao.bytes) || ((kMask & 4) && ac.bytes);
  auto k = bytes ? gather_kernel<kMask, true> : gather_kernel<kMask, false>;
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
