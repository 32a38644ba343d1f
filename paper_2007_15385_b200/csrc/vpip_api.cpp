// vpip_api.cpp -- the reference's C++ API (include/vpip/*.hpp) implemented
// over the B200 C-ABI (include/vpipg.h).
//
// The batch engines and the polygon conversion run on the GPU; the scalar
// early-exit tests, the small geometric helpers and the samplers stay on the
// host, as in the reference (they are not on the batched hot path). Compiled
// with -ffp-contract=off so every host expression rounds like the reference's
// Release build.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <limits>
#include <memory>
#include <mutex>
#include <numbers>
#include <random>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include <cuda_runtime.h>

#include "vpip/engines.hpp"
#include "vpip/error.hpp"
#include "vpip/geometry.hpp"
#include "vpip/sampling.hpp"
#include "vpip/voronoi.hpp"
#include "exact_geom.cuh"
#include "vpipg.h"

namespace vpip {

// ---------------------------------------------------------------- errors
std::string_view error_code_name(ErrorCode code) {
  return vpipg_strerror(static_cast<int>(code) + 1);
}

Error::Error(ErrorCode code, const std::string& message)
    : std::runtime_error(std::string(error_code_name(code)) + ": " + message), code_(code) {}

namespace {

// C-ABI status -> the reference's exception types.
void check(int rc, const char* what) {
  if (rc == 0) return;
  if (rc >= 1 && rc <= 7) throw Error(static_cast<ErrorCode>(rc - 1), what);
  throw std::runtime_error(std::string(what) + ": " + vpipg_strerror(rc));
}

int current_device() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) throw std::runtime_error("vpip: no CUDA device");
  return dev;
}

struct Handle {
  vpipg_poly* p = nullptr;
  ~Handle() { vpipg_destroy(p); }
};

// The batch functions take the polygon / generator set by value semantics on
// every call (engines.hpp:90-142), so a caller looping over batches of one
// polygon would prepare the device tables each time. Prepared handles are
// therefore cached by their exact input (bitwise, per kind and device), 64
// entries, least recently used out; handles are immutable and shared, so a
// cached one may serve concurrent calls (engines.hpp:80-84).
using HandlePtr = std::shared_ptr<Handle>;

HandlePtr cached_handle(int tag, const std::vector<double>& key,
                        const std::function<int(int, vpipg_poly**)>& make, const char* what,
                        int dev) {
  struct Entry {
    int tag, device;
    std::vector<double> key;
    HandlePtr h;
    uint64_t used;
  };
  static std::mutex mu;
  static std::vector<Entry> cache;
  static uint64_t clock = 0;
  {
    std::lock_guard<std::mutex> lock(mu);
    for (Entry& e : cache)
      if (e.tag == tag && e.device == dev && e.key.size() == key.size() &&
          std::memcmp(e.key.data(), key.data(), key.size() * sizeof(double)) == 0) {
        e.used = ++clock;
        return e.h;
      }
  }
  auto h = std::make_shared<Handle>();
  check(make(dev, &h->p), what);  // throws vpip::Error for invalid input
  std::lock_guard<std::mutex> lock(mu);
  if (cache.size() >= 64) {
    auto lru = std::min_element(cache.begin(), cache.end(),
                                [](const Entry& a, const Entry& b) { return a.used < b.used; });
    cache.erase(lru);
  }
  cache.push_back({tag, dev, key, h, ++clock});
  return h;
}

void split(std::span<const Point2> v, std::vector<double>& x, std::vector<double>& y) {
  x.resize(v.size());
  y.resize(v.size());
  for (std::size_t i = 0; i < v.size(); ++i) {
    x[i] = v[i].x;
    y[i] = v[i].y;
  }
}

using Maker = std::function<int(int, vpipg_poly**)>;

// The batch on the B200(s). `threads` keeps the reference's meaning -- how
// many parts the batch is split into, the mask never depending on it
// (test_engines.cpp:227-241) -- and maps to GPUs: with threads > 1 the batch
// is cut into min(threads, devices, m / 2^20) contiguous shards, shard s runs
// on device (current + s) mod devices from its own host thread, each through
// the host-buffer path (one PCIe link per GPU).
InclusionMask run(int engine, const std::vector<double>& key, const Maker& make, const char* what,
                  const PointBatch& points, int threads) {
  if (points.xs.size() != points.ys.size())
    throw Error(ErrorCode::InvalidParameter, "xs and ys differ in length");
  const int dev0 = current_device();
  InclusionMask mask(points.size());
  const size_t m = points.size();
  int ndev = 1;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev < 1) ndev = 1;
  // VPIPG_SHARDS_PER_GPU (default 1) and VPIPG_MIN_SHARD_POINTS (default
  // 2^20) let a single-GPU box exercise the sharded path: several shards per
  // device, run concurrently
  static const int per_gpu = [] {
    const char* v = std::getenv("VPIPG_SHARDS_PER_GPU");
    const int k = v ? std::atoi(v) : 1;
    return k < 1 ? 1 : k;
  }();
  static const size_t min_shard = [] {
    const char* v = std::getenv("VPIPG_MIN_SHARD_POINTS");
    const long long k = v ? std::atoll(v) : (1ll << 20);
    return static_cast<size_t>(k < 1 ? 1 : k);
  }();
  const size_t by_size = std::max<size_t>(1, m / min_shard);
  const int shards = static_cast<int>(std::min<size_t>(
      std::min<size_t>(static_cast<size_t>(std::max(threads, 1)),
                       static_cast<size_t>(ndev) * static_cast<size_t>(per_gpu)),
      by_size));
  // handles first, on the calling thread: validation errors throw from here
  std::vector<HandlePtr> h(shards);
  for (int sh = 0; sh < shards; ++sh) h[sh] = cached_handle(engine, key, make, what, (dev0 + sh) % ndev);
  if (m == 0) return mask;
  if (shards == 1) {
    check(vpipg_test_host(h[0]->p, engine, VPIPG_F64, points.xs.data(), points.ys.data(), m,
                          nullptr, mask.data(), nullptr),
          what);
    return mask;
  }
  std::vector<int> rc(shards, 0);
  std::vector<std::thread> pool;
  const size_t per = (m + shards - 1) / shards;
  for (int sh = 0; sh < shards; ++sh)
    pool.emplace_back([&, sh] {
      const size_t lo = std::min(m, sh * per), hi = std::min(m, lo + per);
      if (lo < hi)
        rc[sh] = vpipg_test_host(h[sh]->p, engine, VPIPG_F64, points.xs.data() + lo,
                                 points.ys.data() + lo, hi - lo, nullptr, mask.data() + lo, nullptr);
    });
  for (auto& t : pool) t.join();
  for (int r : rc) check(r, what);
  return mask;
}

double smin(double a, double b) { return std::min(a, b); }
double smax(double a, double b) { return std::max(a, b); }

}  // namespace

// ---------------------------------------------------------------- geometry
bool Box::valid() const {
  return std::isfinite(min_x) && std::isfinite(min_y) && std::isfinite(max_x) &&
         std::isfinite(max_y) && min_x < max_x && min_y < max_y;
}

Box Box::scaled(double factor) const {
  const Point2 c = center();
  const double hw = 0.5 * factor * width();
  const double hh = 0.5 * factor * height();
  return {c.x - hw, c.y - hh, c.x + hw, c.y + hh};
}

Box bounding_box(std::span<const Point2> points) {
  if (points.empty()) throw Error(ErrorCode::InvalidParameter, "bounding box of an empty point set");
  Box b{points[0].x, points[0].y, points[0].x, points[0].y};
  for (const Point2& p : points) {
    b.min_x = smin(b.min_x, p.x);
    b.min_y = smin(b.min_y, p.y);
    b.max_x = smax(b.max_x, p.x);
    b.max_y = smax(b.max_y, p.y);
  }
  return b;
}

double signed_area(std::span<const Point2> v) {
  double s = 0.0;
  for (std::size_t i = 0, j = v.size() - 1; i < v.size(); j = i++) s += v[j].x * v[i].y - v[i].x * v[j].y;
  return 0.5 * s;
}

double signed_area(const ConvexPolygon& polygon) { return signed_area(polygon.vertices()); }

ConvexPolygon validate_polygon(std::vector<Point2> vertices, double convexity_epsilon) {
  // the checks are exact_geom.cuh's validate_exact, the single definition the
  // C-ABI prepare and the device CSR ingest also run
  const int n = static_cast<int>(vertices.size());
  bool reversed = false;
  int at = -1;
  const int rc = vpipg::validate_exact(
      [&](int k) { return make_double2(vertices[k].x, vertices[k].y); }, n, &reversed,
      convexity_epsilon, &at);
  switch (rc) {
    case 0: break;
    case 4: throw Error(ErrorCode::NonFinite, "vertex " + std::to_string(at));
    case 1: throw Error(ErrorCode::TooFewVertices, std::to_string(n) + " vertices");
    case 3:
      throw Error(ErrorCode::DegenerateEdge,
                  "vertices " + std::to_string((at + n - 1) % n) + " and " + std::to_string(at));
    default:
      throw Error(ErrorCode::NotConvex, at >= 0 ? "collinear or reflex vertex at index " + std::to_string(at)
                                                : std::string("winds more than once"));
  }
  if (reversed) std::reverse(vertices.begin(), vertices.end());
  return ConvexPolygon(std::move(vertices), reversed);
}

Point2 centroid(const ConvexPolygon& polygon) { return to_voronoi(polygon).inner; }

// ---------------------------------------------------------------- voronoi helpers
EdgeCoefficients edge_coefficients(Point2 qi, Point2 qj, double degenerate_sq) {
  const double a = qi.y - qj.y;
  const double b = qj.x - qi.x;
  const double c = -(a * qi.x + b * qi.y);
  if (a * a + b * b <= degenerate_sq) throw Error(ErrorCode::DegenerateEdge, "edge endpoints coincide");
  return {a, b, c};
}

double line_distance(const EdgeCoefficients& e, Point2 p) {
  return std::abs(e.a * p.x + e.b * p.y + e.c) / std::hypot(e.a, e.b);
}

Point2 foot_of_perpendicular(Point2 p0, const EdgeCoefficients& e) {
  const double d = e.a * e.a + e.b * e.b;
  return {(e.b * e.b * p0.x - e.a * e.b * p0.y - e.c * e.a) / d,
          (-e.a * e.b * p0.x + e.a * e.a * p0.y - e.c * e.b) / d};
}

Point2 reflect_generator(Point2 p0, const EdgeCoefficients& e, double collision_rel) {
  const double a = e.a, b = e.b, d = a * a + b * b;
  if (std::abs(a * p0.x + b * p0.y + e.c) <= collision_rel * d)
    throw Error(ErrorCode::GeneratorCollision, "point lies on the edge line");
  return {((b * b - a * a) * p0.x - 2.0 * a * b * p0.y - 2.0 * e.c * a) / d,
          (-2.0 * a * b * p0.x + (a * a - b * b) * p0.y - 2.0 * e.c * b) / d};
}

GeneratorSet to_voronoi(const ConvexPolygon& polygon) {
  std::vector<double> x, y;
  split(polygon.vertices(), x, y);
  Handle h;
  check(vpipg_prepare(x.data(), y.data(), static_cast<uint32_t>(x.size()), VPIPG_KIND_VORONOI,
                      current_device(), nullptr, &h.p),
        "to_voronoi");
  std::vector<double> outer(2 * x.size());
  double inner[2];
  check(vpipg_poly_generators(h.p, inner, outer.data()), "to_voronoi");
  GeneratorSet g;
  g.inner = {inner[0], inner[1]};
  g.outer.resize(x.size());
  for (std::size_t k = 0; k < x.size(); ++k) g.outer[k] = {outer[2 * k], outer[2 * k + 1]};
  return g;
}

double edge_line_distance(const ConvexPolygon& polygon, Point2 p) {
  const auto v = polygon.vertices();
  double nearest = std::numeric_limits<double>::infinity();
  for (std::size_t k = 0; k < v.size(); ++k)
    nearest = smin(nearest, line_distance(edge_coefficients(v[k], v[(k + 1) % v.size()]), p));
  return nearest;
}

// ---------------------------------------------------------------- engines
PointBatch PointBatch::from_points(std::span<const Point2> points) {
  PointBatch b;
  b.reserve(points.size());
  for (const Point2& p : points) b.push_back(p);
  return b;
}

std::size_t count_inside(const InclusionMask& mask) {
  std::size_t s = 0;
  for (std::uint8_t b : mask) s += b;
  return s;
}

std::string_view engine_name(EngineKind kind) {
  switch (kind) {
    case EngineKind::Voronoi: return "voronoi";
    case EngineKind::SignOfOffset: return "sign_of_offset";
    case EngineKind::RayCrossing: return "ray_crossing";
  }
  return "unknown";
}

std::optional<EngineKind> parse_engine(std::string_view name) {
  if (name == "voronoi") return EngineKind::Voronoi;
  if (name == "sign_of_offset" || name == "offset") return EngineKind::SignOfOffset;
  if (name == "ray_crossing" || name == "crossing") return EngineKind::RayCrossing;
  return std::nullopt;
}

bool voronoi_contains(const GeneratorSet& g, Point2 p) {
  const double inner_sq = squared_distance(p, g.inner);
  for (const Point2& o : g.outer)
    if (squared_distance(p, o) < inner_sq) return false;
  return true;
}

InclusionMask voronoi_contains_batch(const GeneratorSet& g, const PointBatch& points, int threads) {
  std::vector<double> outer(2 * g.outer.size());
  for (std::size_t k = 0; k < g.outer.size(); ++k) {
    outer[2 * k] = g.outer[k].x;
    outer[2 * k + 1] = g.outer[k].y;
  }
  const double inner[2] = {g.inner.x, g.inner.y};
  std::vector<double> key(outer);
  key.push_back(inner[0]);
  key.push_back(inner[1]);
  return run(
      VPIPG_ENGINE_VORONOI, key,
      [&](int dev, vpipg_poly** out) {
        return vpipg_prepare_generators(inner, outer.data(), static_cast<uint32_t>(g.outer.size()),
                                        dev, nullptr, out);
      },
      "voronoi_contains_batch", points, threads);
}

InclusionMask voronoi_contains_batch(const GeneratorSet& g, const PointBatch& points,
                                     BatchStats& stats, int threads) {
  InclusionMask mask = voronoi_contains_batch(g, points, threads);
  // the device kernel is branch-free: (n+1)*m evaluations, n*m comparisons
  stats.distance_evaluations += (g.edge_count() + 1) * points.size();
  stats.comparisons += g.edge_count() * points.size();
  return mask;
}

InclusionMask voronoi_contains_batch_sqrt(const GeneratorSet& g, const PointBatch& points, int) {
  InclusionMask mask(points.size());
  for (std::size_t j = 0; j < points.size(); ++j) {
    const double inner = std::sqrt(squared_distance(points.at(j), g.inner));
    std::uint8_t in = 1;
    for (const Point2& o : g.outer) in &= static_cast<std::uint8_t>(inner <= std::sqrt(squared_distance(points.at(j), o)));
    mask[j] = in;
  }
  return mask;
}

SquaredDistanceTable squared_distance_table(const GeneratorSet& g, const PointBatch& points) {
  const std::size_t rows = g.edge_count() + 1, cols = points.size();
  SquaredDistanceTable t{rows, cols, std::vector<double>(rows * cols)};
  for (std::size_t r = 0; r < rows; ++r) {
    const Point2 q = r == 0 ? g.inner : g.outer[r - 1];
    for (std::size_t j = 0; j < cols; ++j) t.values[r * cols + j] = squared_distance(points.at(j), q);
  }
  return t;
}

bool sign_of_offset_contains(const ConvexPolygon& polygon, Point2 p) {
  const auto v = polygon.vertices();
  for (std::size_t i = 0, j = v.size() - 1; i < v.size(); j = i++) {
    const double dvx = v[i].x - v[j].x, dvy = v[i].y - v[j].y;
    if (p.y * dvx - p.x * dvy < v[j].y * dvx - v[j].x * dvy) return false;
  }
  return true;
}

InclusionMask sign_of_offset_contains_batch(const ConvexPolygon& polygon, const PointBatch& points,
                                            int threads) {
  std::vector<double> x, y;
  split(polygon.vertices(), x, y);
  std::vector<double> key(x);
  key.insert(key.end(), y.begin(), y.end());
  return run(
      VPIPG_ENGINE_OFFSET, key,
      [&](int dev, vpipg_poly** out) {
        return vpipg_prepare(x.data(), y.data(), static_cast<uint32_t>(x.size()), VPIPG_KIND_OFFSET, dev,
                             nullptr, out);
      },
      "sign_of_offset_contains_batch", points, threads);
}

namespace {
bool on_segment_or_cross(Point2 w, Point2 u, Point2 p, int& crossings) {
  const double dvx = u.x - w.x, dvy = u.y - w.y;
  const bool in_range = (u.y > p.y) != (w.y > p.y);
  const double lhs = p.y * dvx - p.x * dvy;
  const double rhs = w.y * dvx - w.x * dvy;
  crossings += in_range && (lhs != rhs) && ((lhs > rhs) == (u.y > w.y));
  return lhs == rhs && p.x >= smin(w.x, u.x) && p.x <= smax(w.x, u.x) && p.y >= smin(w.y, u.y) &&
         p.y <= smax(w.y, u.y);
}
}  // namespace

bool ray_crossing_contains(std::span<const Point2> v, Point2 p) {
  int crossings = 0;
  for (std::size_t i = 0, j = v.size() - 1; i < v.size(); j = i++)
    if (on_segment_or_cross(v[j], v[i], p, crossings)) return true;
  return (crossings & 1) != 0;
}

int ray_crossing_count(std::span<const Point2> v, Point2 p) {
  int crossings = 0;
  for (std::size_t i = 0, j = v.size() - 1; i < v.size(); j = i++) on_segment_or_cross(v[j], v[i], p, crossings);
  return crossings;
}

InclusionMask ray_crossing_contains_batch(std::span<const Point2> vertices, const PointBatch& points,
                                          int threads) {
  std::vector<double> x, y;
  split(vertices, x, y);
  std::vector<double> key(x);
  key.insert(key.end(), y.begin(), y.end());
  return run(
      VPIPG_ENGINE_CROSSING, key,
      [&](int dev, vpipg_poly** out) {
        return vpipg_prepare(x.data(), y.data(), static_cast<uint32_t>(x.size()), VPIPG_KIND_CROSSING, dev,
                             nullptr, out);
      },
      "ray_crossing_contains_batch", points, threads);
}

// ---------------------------------------------------------------- sampling
namespace {
double unit_real(std::mt19937_64& rng) { return static_cast<double>(rng() >> 11) * 0x1.0p-53; }
void check_params(std::size_t n, double r, Point2 c) {
  if (n < 3) throw Error(ErrorCode::InvalidParameter, "polygon needs at least 3 vertices");
  if (!std::isfinite(r) || r <= 0.0) throw Error(ErrorCode::InvalidParameter, "circumradius must be positive and finite");
  if (!is_finite(c)) throw Error(ErrorCode::InvalidParameter, "center must be finite");
}
}  // namespace

ConvexPolygon regular_polygon(std::size_t n, double r, Point2 c) {
  check_params(n, r, c);
  std::vector<Point2> v(n);
  for (std::size_t k = 0; k < n; ++k) {
    const double a = 2.0 * std::numbers::pi * static_cast<double>(k) / static_cast<double>(n) +
                     std::numbers::pi / 2.0;
    v[k] = {c.x + r * std::cos(a), c.y + r * std::sin(a)};
  }
  return validate_polygon(std::move(v));
}

ConvexPolygon random_convex_polygon(std::size_t n, std::uint64_t seed, double r, Point2 c) {
  check_params(n, r, c);
  std::mt19937_64 rng(seed);
  const double min_gap = 2.0 * std::numbers::pi / (20.0 * static_cast<double>(n));
  std::vector<double> ang(n);
  for (int attempt = 0; attempt < 1024; ++attempt) {
    for (double& a : ang) a = 2.0 * std::numbers::pi * unit_real(rng);
    std::sort(ang.begin(), ang.end());
    bool ok = ang.front() + 2.0 * std::numbers::pi - ang.back() >= min_gap;
    for (std::size_t k = 1; ok && k < n; ++k) ok = ang[k] - ang[k - 1] >= min_gap;
    if (!ok) continue;
    std::vector<Point2> v(n);
    for (std::size_t k = 0; k < n; ++k) v[k] = {c.x + r * std::cos(ang[k]), c.y + r * std::sin(ang[k])};
    return validate_polygon(std::move(v));
  }
  throw Error(ErrorCode::InvalidParameter, "no well-spaced angle draw after 1024 attempts");
}

PointBatch sample_points(std::size_t count, const Box& box, std::uint64_t seed) {
  if (!box.valid()) throw Error(ErrorCode::InvalidParameter, "sampling box is degenerate");
  std::mt19937_64 rng(seed);
  PointBatch b;
  b.xs.resize(count);
  b.ys.resize(count);
  const double w = box.width(), h = box.height();
  for (std::size_t j = 0; j < count; ++j) {
    b.xs[j] = box.min_x + w * unit_real(rng);
    b.ys[j] = box.min_y + h * unit_real(rng);
  }
  return b;
}

std::uint64_t mix_seed(std::uint64_t seed, std::uint64_t salt) { return vpipg_mix_seed(seed, salt); }

}  // namespace vpip

// ---------------------------------------------------------------- C-ABI samplers
extern "C" {

uint64_t vpipg_mix_seed(uint64_t seed, uint64_t salt) { return vpipg::mix_seed(seed, salt); }

static int sampler_status(const vpip::Error& e) { return static_cast<int>(e.code()) + 1; }

static void copy_out(const vpip::ConvexPolygon& p, double* vx, double* vy) {
  for (std::size_t i = 0; i < p.size(); ++i) {
    vx[i] = p.vertex(i).x;
    vy[i] = p.vertex(i).y;
  }
}

int vpipg_regular_polygon(uint32_t n, double r, double cx, double cy, double* vx, double* vy) {
  try {
    copy_out(vpip::regular_polygon(n, r, {cx, cy}), vx, vy);
    return 0;
  } catch (const vpip::Error& e) {
    return sampler_status(e);
  }
}

int vpipg_random_convex_polygon(uint32_t n, uint64_t seed, double r, double cx, double cy,
                                double* vx, double* vy) {
  try {
    copy_out(vpip::random_convex_polygon(n, seed, r, {cx, cy}), vx, vy);
    return 0;
  } catch (const vpip::Error& e) {
    return sampler_status(e);
  }
}

int vpipg_sample_points(uint64_t count, double min_x, double min_y, double max_x, double max_y,
                        uint64_t seed, double* xs, double* ys) {
  try {
    const vpip::PointBatch b = vpip::sample_points(count, {min_x, min_y, max_x, max_y}, seed);
    std::memcpy(xs, b.xs.data(), count * sizeof(double));
    std::memcpy(ys, b.ys.data(), count * sizeof(double));
    return 0;
  } catch (const vpip::Error& e) {
    return sampler_status(e);
  }
}

}  // extern "C"
