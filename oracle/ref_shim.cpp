// ref_shim.cpp -- extern "C" access to the UNMODIFIED reference library.
//
// TEST INFRASTRUCTURE ONLY. oracle/Makefile compiles the reference's own
// sources where they lie (/root/reference/proj/src/{geometry,voronoi,engines,
// sampling}.cpp) together with this file into oracle/_ref/libvpip_ref.so.
// It is used (a) to pin the C restatement (oracle/vpip_oracle.c) against the
// reference itself, (b) to generate tests/golden/ fixtures, and (c) as the
// CPU baseline arm of bench.py (`--impl reference`, cpu_baseline.kind =
// "reference"). Nothing here is on the product path.
#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <optional>
#include <sstream>
#include <thread>
#include <vector>

#include "vpip/bench.hpp"
#include "vpip/engines.hpp"
#include "vpip/geometry.hpp"
#include "vpip/sampling.hpp"
#include "vpip/voronoi.hpp"

namespace {

std::vector<vpip::Point2> to_points(const double* vx, const double* vy, std::size_t n) {
  std::vector<vpip::Point2> v(n);
  for (std::size_t i = 0; i < n; ++i) v[i] = {vx[i], vy[i]};
  return v;
}

int code_of(const vpip::Error& e) { return static_cast<int>(e.code()) + 1; }

struct Poly {
  std::vector<vpip::Point2> raw;              // as given (crossing engine input)
  std::optional<vpip::ConvexPolygon> convex;  // validated (voronoi / offset)
  std::optional<vpip::GeneratorSet> gens;
};

}  // namespace

extern "C" {

int vr_validate(const double* vx, const double* vy, std::size_t n, double* ox, double* oy,
                int* reversed) {
  try {
    vpip::ConvexPolygon p = vpip::validate_polygon(to_points(vx, vy, n));
    for (std::size_t i = 0; i < p.size(); ++i) {
      ox[i] = p.vertex(i).x;
      oy[i] = p.vertex(i).y;
    }
    *reversed = p.was_reversed() ? 1 : 0;
    return 0;
  } catch (const vpip::Error& e) {
    return code_of(e);
  }
}

int vr_to_voronoi(const double* vx, const double* vy, std::size_t n, double* inner_xy,
                  double* outer_xy) {
  try {
    const vpip::GeneratorSet g = vpip::to_voronoi(vpip::validate_polygon(to_points(vx, vy, n)));
    inner_xy[0] = g.inner.x;
    inner_xy[1] = g.inner.y;
    for (std::size_t k = 0; k < g.outer.size(); ++k) {
      outer_xy[2 * k] = g.outer[k].x;
      outer_xy[2 * k + 1] = g.outer[k].y;
    }
    return 0;
  } catch (const vpip::Error& e) {
    return code_of(e);
  }
}

int vr_edge_coefficients(double qix, double qiy, double qjx, double qjy, double* abc) {
  try {
    const vpip::EdgeCoefficients e = vpip::edge_coefficients({qix, qiy}, {qjx, qjy});
    abc[0] = e.a;
    abc[1] = e.b;
    abc[2] = e.c;
    return 0;
  } catch (const vpip::Error& e) {
    return code_of(e);
  }
}

int vr_reflect_generator(double px, double py, const double* abc, double* r) {
  try {
    const vpip::Point2 q = vpip::reflect_generator({px, py}, {abc[0], abc[1], abc[2]});
    r[0] = q.x;
    r[1] = q.y;
    return 0;
  } catch (const vpip::Error& e) {
    return code_of(e);
  }
}

double vr_edge_line_distance(const double* vx, const double* vy, std::size_t n, double px,
                             double py) {
  return vpip::edge_line_distance(vpip::validate_polygon(to_points(vx, vy, n)), {px, py});
}

uint64_t vr_mix_seed(uint64_t seed, uint64_t salt) { return vpip::mix_seed(seed, salt); }

int vr_sample_points(std::size_t count, double min_x, double min_y, double max_x, double max_y,
                     uint64_t seed, double* xs, double* ys) {
  try {
    const vpip::PointBatch b = vpip::sample_points(count, {min_x, min_y, max_x, max_y}, seed);
    std::memcpy(xs, b.xs.data(), count * sizeof(double));
    std::memcpy(ys, b.ys.data(), count * sizeof(double));
    return 0;
  } catch (const vpip::Error& e) {
    return code_of(e);
  }
}

int vr_regular_polygon(std::size_t n, double r, double cx, double cy, double* vx, double* vy) {
  try {
    const vpip::ConvexPolygon p = vpip::regular_polygon(n, r, {cx, cy});
    for (std::size_t i = 0; i < n; ++i) {
      vx[i] = p.vertex(i).x;
      vy[i] = p.vertex(i).y;
    }
    return 0;
  } catch (const vpip::Error& e) {
    return code_of(e);
  }
}

int vr_random_convex_polygon(std::size_t n, uint64_t seed, double r, double cx, double cy,
                             double* vx, double* vy) {
  try {
    const vpip::ConvexPolygon p = vpip::random_convex_polygon(n, seed, r, {cx, cy});
    for (std::size_t i = 0; i < n; ++i) {
      vx[i] = p.vertex(i).x;
      vy[i] = p.vertex(i).y;
    }
    return 0;
  } catch (const vpip::Error& e) {
    return code_of(e);
  }
}

// ---- batch engines through opaque handles (input copies are untimed) ----

void* vr_batch_new(const double* xs, const double* ys, std::size_t m) {
  auto* b = new vpip::PointBatch;
  b->xs.assign(xs, xs + m);
  b->ys.assign(ys, ys + m);
  return b;
}

void vr_batch_free(void* b) { delete static_cast<vpip::PointBatch*>(b); }

// Builds the engine inputs the way the reference CLI does (vpip.cpp:120-133):
// raw vertices for crossing, validate + to_voronoi for the others. Returns
// nullptr and sets *code when validation or conversion throws.
void* vr_poly_new(const double* vx, const double* vy, std::size_t n, int want_convex, int* code) {
  auto* p = new Poly;
  p->raw = to_points(vx, vy, n);
  *code = 0;
  if (want_convex) {
    try {
      p->convex.emplace(vpip::validate_polygon(p->raw));
      p->gens.emplace(vpip::to_voronoi(*p->convex));
    } catch (const vpip::Error& e) {
      *code = code_of(e);
      delete p;
      return nullptr;
    }
  }
  return p;
}

void vr_poly_free(void* p) { delete static_cast<Poly*>(p); }

// engine: 0 voronoi, 1 sign_of_offset, 2 ray_crossing (vpip::EngineKind order).
// Times only the *_contains_batch call, as run_benchmark does
// (bench.cpp:196-199); copies the byte mask out afterwards when out != null.
int vr_run_engine(void* poly, int engine, void* batch, int threads, uint8_t* out,
                  uint64_t* ns, uint64_t* inside) {
  const Poly& p = *static_cast<Poly*>(poly);
  const vpip::PointBatch& b = *static_cast<vpip::PointBatch*>(batch);
  if (engine != 2 && !p.convex) return 6;
  vpip::InclusionMask mask;
  const auto t0 = std::chrono::steady_clock::now();
  switch (engine) {
    case 0: mask = vpip::voronoi_contains_batch(*p.gens, b, threads); break;
    case 1: mask = vpip::sign_of_offset_contains_batch(*p.convex, b, threads); break;
    case 2: mask = vpip::ray_crossing_contains_batch(p.raw, b, threads); break;
    default: return 6;
  }
  const auto t1 = std::chrono::steady_clock::now();
  if (ns) *ns = static_cast<uint64_t>(std::chrono::duration_cast<std::chrono::nanoseconds>(t1 - t0).count());
  if (inside) *inside = vpip::count_inside(mask);
  if (out) std::memcpy(out, mask.data(), mask.size());
  return 0;
}

// Voronoi batch on an explicit generator set (any GeneratorSet, e.g. one
// read back from the GPU), plus the instrumented work counters.
void vr_voronoi_batch_gens(const double* inner_xy, const double* outer_xy, std::size_t n,
                           void* batch, int threads, uint8_t* out, uint64_t* evals,
                           uint64_t* comps) {
  vpip::GeneratorSet g;
  g.inner = {inner_xy[0], inner_xy[1]};
  for (std::size_t k = 0; k < n; ++k) g.outer.push_back({outer_xy[2 * k], outer_xy[2 * k + 1]});
  vpip::BatchStats stats;
  const vpip::InclusionMask mask =
      vpip::voronoi_contains_batch(g, *static_cast<vpip::PointBatch*>(batch), stats, threads);
  std::memcpy(out, mask.data(), mask.size());
  if (evals) *evals = stats.distance_evaluations;
  if (comps) *comps = stats.comparisons;
}

// ---- polygon-database join baseline (config 4) ----
// The reference has no gather API; its natural use is one batch call per
// polygon over that polygon's points. vr_join_new groups the
// pairs by id and validates / converts every polygon (untimed preparation);
// vr_join_run times the per-polygon *_contains_batch calls, polygons split
// over `threads` std::threads, each call single-threaded.
struct Join {
  std::vector<Poly> polys;
  std::vector<vpip::PointBatch> batches;
  std::vector<std::vector<std::uint64_t>> index;
};

void* vr_join_new(const uint32_t* offsets, const double* vx, const double* vy, uint32_t npoly,
                  const double* xs, const double* ys, const uint32_t* ids, std::size_t m) {
  auto* j = new Join;
  j->polys.resize(npoly);
  j->batches.resize(npoly);
  j->index.resize(npoly);
  for (uint32_t i = 0; i < npoly; ++i) {
    Poly& p = j->polys[i];
    p.raw = to_points(vx + offsets[i], vy + offsets[i], offsets[i + 1] - offsets[i]);
    try {
      p.convex.emplace(vpip::validate_polygon(p.raw));
      p.gens.emplace(vpip::to_voronoi(*p.convex));
    } catch (const vpip::Error&) {
    }
  }
  for (std::size_t k = 0; k < m; ++k) {
    if (ids[k] >= npoly) continue;
    j->batches[ids[k]].push_back({xs[k], ys[k]});
    j->index[ids[k]].push_back(k);
  }
  return j;
}

void vr_join_free(void* j) { delete static_cast<Join*>(j); }

uint64_t vr_join_run(void* jp, int engine, int threads, uint8_t* out) {
  Join& j = *static_cast<Join*>(jp);
  const std::size_t np = j.polys.size();
  std::vector<vpip::InclusionMask> masks(np);
  auto work = [&](std::size_t lo, std::size_t hi) {
    for (std::size_t i = lo; i < hi; ++i) {
      const Poly& p = j.polys[i];
      const vpip::PointBatch& b = j.batches[i];
      if (b.empty()) continue;
      if (engine == 2) masks[i] = vpip::ray_crossing_contains_batch(p.raw, b, 1);
      else if (!p.convex) masks[i].assign(b.size(), 0);
      else if (engine == 0) masks[i] = vpip::voronoi_contains_batch(*p.gens, b, 1);
      else masks[i] = vpip::sign_of_offset_contains_batch(*p.convex, b, 1);
    }
  };
  const auto t0 = std::chrono::steady_clock::now();
  {
    std::vector<std::jthread> pool;
    const int t = std::max(threads, 1);
    for (int c = 0; c < t; ++c) pool.emplace_back(work, np * c / t, np * (c + 1) / t);
  }
  const auto t1 = std::chrono::steady_clock::now();
  if (out)
    for (std::size_t i = 0; i < np; ++i)
      for (std::size_t k = 0; k < masks[i].size(); ++k) out[j.index[i][k]] = masks[i][k];
  return static_cast<uint64_t>(std::chrono::duration_cast<std::chrono::nanoseconds>(t1 - t0).count());
}

// run_validation (bench.cpp:279-308) on a convex polygon handle: fills
// counts[0..4] = {v/o, v/c, o/c pair disagreements, disagreeing points, pass}.
int vr_run_validation(void* poly, void* batch, int threads, double band, uint64_t* counts) {
  const Poly& p = *static_cast<Poly*>(poly);
  if (!p.convex) return 6;
  const vpip::ValidationReport r = vpip::run_validation(
      *p.convex, *p.gens, *static_cast<vpip::PointBatch*>(batch), threads, band);
  for (int i = 0; i < 3; ++i) counts[i] = r.pair_disagreements[i];
  counts[3] = r.disagreeing_points;
  counts[4] = r.pass ? 1 : 0;
  return 0;
}

// read_bench_csv (bench.cpp:177-208) on a CSV text; returns the record count
// (or -1 on a parse error) and the median Query wall time per (engine, n) in
// `medians` laid out [engine][n - 3] for n = 3..15 (0 when absent).
long vr_read_bench_csv(const char* text, double* medians) {
  try {
    std::istringstream in(text);
    const std::vector<vpip::BenchRecord> recs = vpip::read_bench_csv(in);
    std::vector<double> t[3][13];
    for (const vpip::BenchRecord& r : recs)
      if (r.phase == vpip::BenchPhase::Query && r.n_edges >= 3 && r.n_edges <= 15)
        t[static_cast<int>(r.engine)][r.n_edges - 3].push_back(static_cast<double>(r.wall_time_ns));
    for (int e = 0; e < 3; ++e)
      for (int i = 0; i < 13; ++i) medians[e * 13 + i] = t[e][i].empty() ? 0.0 : vpip::median(t[e][i]);
    return static_cast<long>(recs.size());
  } catch (const vpip::Error&) {
    return -1;
  }
}

// ---- full-size runs in chunks (bench.py's CPU legs) ----
// A workload of m f32 points (BASELINE C5 is 2^31 points, 32 GiB as the
// reference's f64 PointBatch) is held as PointBatch chunks of <= `chunk`
// points, widened from f32 once (untimed, in parallel). vr_chunked_run then
// runs one engine over every chunk exactly as run_benchmark times a batch
// call (bench.cpp:196-199): only the *_contains_batch call is in `ns`;
// count_inside (engines.cpp:215-217) is timed as its own step (`count_ns`);
// the byte mask is packed LSB-first into `packed` (io.cpp:272-279 order)
// outside both timings.
void* vr_chunks_new(const float* xs, const float* ys, std::size_t m, std::size_t chunk, int threads) {
  auto* v = new std::vector<vpip::PointBatch>((m + chunk - 1) / chunk);
  auto work = [&](std::size_t c0, std::size_t c1) {
    for (std::size_t c = c0; c < c1; ++c) {
      const std::size_t lo = c * chunk, hi = std::min(m, lo + chunk);
      vpip::PointBatch& b = (*v)[c];
      b.xs.resize(hi - lo);
      b.ys.resize(hi - lo);
      for (std::size_t i = lo; i < hi; ++i) {
        b.xs[i - lo] = static_cast<double>(xs[i]);
        b.ys[i - lo] = static_cast<double>(ys[i]);
      }
    }
  };
  const std::size_t nc = v->size();
  const int t = std::max(1, std::min<int>(threads, static_cast<int>(nc)));
  {
    std::vector<std::jthread> pool;
    for (int i = 0; i < t; ++i) pool.emplace_back(work, nc * i / t, nc * (i + 1) / t);
  }
  return v;
}

void vr_chunks_free(void* v) { delete static_cast<std::vector<vpip::PointBatch>*>(v); }

int vr_chunked_run(void* poly, void* chunks, int engine, int threads, uint8_t* packed, uint64_t* ns,
                   uint64_t* count_ns, uint64_t* inside) {
  const Poly& p = *static_cast<Poly*>(poly);
  if (engine != 2 && !p.convex) return 6;
  uint64_t t_run = 0, t_cnt = 0, total = 0, base = 0;
  for (const vpip::PointBatch& b : *static_cast<std::vector<vpip::PointBatch>*>(chunks)) {
    vpip::InclusionMask mask;
    const auto t0 = std::chrono::steady_clock::now();
    switch (engine) {
      case 0: mask = vpip::voronoi_contains_batch(*p.gens, b, threads); break;
      case 1: mask = vpip::sign_of_offset_contains_batch(*p.convex, b, threads); break;
      case 2: mask = vpip::ray_crossing_contains_batch(p.raw, b, threads); break;
      default: return 6;
    }
    const auto t1 = std::chrono::steady_clock::now();
    total += vpip::count_inside(mask);
    const auto t2 = std::chrono::steady_clock::now();
    t_run += static_cast<uint64_t>(std::chrono::duration_cast<std::chrono::nanoseconds>(t1 - t0).count());
    t_cnt += static_cast<uint64_t>(std::chrono::duration_cast<std::chrono::nanoseconds>(t2 - t1).count());
    if (packed) {  // chunks are multiples of 8 points except the last
      for (std::size_t i = 0; i < mask.size(); ++i)
        if (mask[i]) packed[(base + i) >> 3] |= static_cast<uint8_t>(1u << ((base + i) & 7));
    }
    base += mask.size();
  }
  if (ns) *ns = t_run;
  if (count_ns) *count_ns = t_cnt;
  if (inside) *inside = total;
  return 0;
}

// The per-pair scalar join ("also report the per-pair
// scalar loop"): the reference's early-exit scalar tests (engines.cpp:235-241,
// :304-318, :331-350) on every pair in stream order, i.e. random polygon ids,
// pairs split over `threads` std::threads. Returns ns; fills the byte mask.
uint64_t vr_join_scalar(void* jp, const double* xs, const double* ys, const uint32_t* ids,
                        std::size_t m, int engine, int threads, uint8_t* out) {
  Join& j = *static_cast<Join*>(jp);
  const uint32_t np = static_cast<uint32_t>(j.polys.size());
  auto work = [&](std::size_t lo, std::size_t hi) {
    for (std::size_t k = lo; k < hi; ++k) {
      uint8_t r = 0;
      if (ids[k] < np) {
        const Poly& p = j.polys[ids[k]];
        const vpip::Point2 q{xs[k], ys[k]};
        if (engine == 2) r = vpip::ray_crossing_contains(p.raw, q);
        else if (p.convex) r = engine == 0 ? vpip::voronoi_contains(*p.gens, q)
                                           : vpip::sign_of_offset_contains(*p.convex, q);
      }
      out[k] = r;
    }
  };
  const auto t0 = std::chrono::steady_clock::now();
  {
    std::vector<std::jthread> pool;
    const int t = std::max(threads, 1);
    for (int c = 0; c < t; ++c) pool.emplace_back(work, m * c / t, m * (c + 1) / t);
  }
  const auto t1 = std::chrono::steady_clock::now();
  return static_cast<uint64_t>(std::chrono::duration_cast<std::chrono::nanoseconds>(t1 - t0).count());
}

// The conversion phase of run_benchmark (bench.cpp:165-170: to_voronoi of an
// already validated polygon) and, separately, validate_polygon
// (geometry.cpp:53-98): medians over `reps` calls, ns. Returns 0 or the code.
int vr_time_convert(const double* vx, const double* vy, std::size_t n, int reps,
                    uint64_t* ns_validate, uint64_t* ns_convert) {
  try {
    const std::vector<vpip::Point2> raw = to_points(vx, vy, n);
    std::vector<uint64_t> tv, tc;
    uint64_t sink = 0;
    for (int r = 0; r < reps; ++r) {
      const auto t0 = std::chrono::steady_clock::now();
      const vpip::ConvexPolygon p = vpip::validate_polygon(raw);
      const auto t1 = std::chrono::steady_clock::now();
      const vpip::GeneratorSet g = vpip::to_voronoi(p);
      const auto t2 = std::chrono::steady_clock::now();
      sink += g.outer.size();
      tv.push_back(std::chrono::duration_cast<std::chrono::nanoseconds>(t1 - t0).count());
      tc.push_back(std::chrono::duration_cast<std::chrono::nanoseconds>(t2 - t1).count());
    }
    std::sort(tv.begin(), tv.end());
    std::sort(tc.begin(), tc.end());
    *ns_validate = tv[tv.size() / 2] + (sink == 0 ? 1 : 0);
    *ns_convert = tc[tc.size() / 2];
    return 0;
  } catch (const vpip::Error& e) {
    return code_of(e);
  }
}

// The same phases over a CSR polygon database, one thread, all polygons:
// total ns of validate_polygon and of to_voronoi (failures skip to_voronoi).
void vr_time_convert_csr(const uint32_t* offsets, const double* vx, const double* vy,
                         uint32_t npoly, uint64_t* ns_validate, uint64_t* ns_convert) {
  uint64_t tv = 0, tc = 0, sink = 0;
  for (uint32_t i = 0; i < npoly; ++i) {
    const std::vector<vpip::Point2> raw =
        to_points(vx + offsets[i], vy + offsets[i], offsets[i + 1] - offsets[i]);
    const auto t0 = std::chrono::steady_clock::now();
    std::optional<vpip::ConvexPolygon> p;
    try {
      p.emplace(vpip::validate_polygon(raw));
    } catch (const vpip::Error&) {
    }
    const auto t1 = std::chrono::steady_clock::now();
    tv += std::chrono::duration_cast<std::chrono::nanoseconds>(t1 - t0).count();
    if (p) {
      try {
        sink += vpip::to_voronoi(*p).outer.size();
      } catch (const vpip::Error&) {
      }
      tc += std::chrono::duration_cast<std::chrono::nanoseconds>(std::chrono::steady_clock::now() - t1).count();
    }
  }
  *ns_validate = tv + (sink == 0 ? 1 : 0);
  *ns_convert = tc;
}

int vr_scalar(void* poly, int engine, double px, double py) {
  const Poly& p = *static_cast<Poly*>(poly);
  switch (engine) {
    case 0: return vpip::voronoi_contains(*p.gens, {px, py});
    case 1: return vpip::sign_of_offset_contains(*p.convex, {px, py});
    case 2: return vpip::ray_crossing_contains(p.raw, {px, py});
    case 3: return vpip::ray_crossing_count(p.raw, {px, py});
    default: return -1;
  }
}

}  // extern "C"
