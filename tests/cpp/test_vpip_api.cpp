// test_vpip_api.cpp -- the vpip:: C++ drop-in (include/vpip/) on the GPU.
//
// Re-expresses the reference's doctest known answers (proj/tests/
// test_engines.cpp, test_voronoi.cpp, test_geometry.cpp) and acceptance
// criteria 1, 5, 7, 8 (proj/tests/acceptance.cpp) against the B200 engine
// through the unchanged C++ signatures. Exit code 0 iff every check holds.
#include <cmath>
#include <cstdio>
#include <functional>
#include <thread>
#include <vector>

#include "vpip/engines.hpp"
#include "vpip/geometry.hpp"
#include "vpip/sampling.hpp"
#include "vpip/voronoi.hpp"

using namespace vpip;

static int g_fail = 0, g_checks = 0;
#define CHECK(cond)                                                     \
  do {                                                                  \
    ++g_checks;                                                         \
    if (!(cond)) {                                                      \
      ++g_fail;                                                         \
      std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond);       \
    }                                                                   \
  } while (0)

template <class F>
static int thrown_code(F f) {
  try {
    f();
  } catch (const Error& e) {
    return static_cast<int>(e.code());
  }
  return -1;
}

static ConvexPolygon unit_square() { return validate_polygon({{0, 0}, {1, 0}, {1, 1}, {0, 1}}); }

static ConvexPolygon make_test_polygon(std::uint64_t i) {  // test_engines.cpp:32-38
  const std::size_t n = 3 + static_cast<std::size_t>(mix_seed(21, i) % 13);
  const double radius = 0.5 + 2.0 * static_cast<double>(mix_seed(22, i) % 100) / 100.0;
  const Point2 c = {static_cast<double>(mix_seed(23, i) % 7) - 3.0,
                    static_cast<double>(mix_seed(24, i) % 7) - 3.0};
  return random_convex_polygon(n, mix_seed(25, i), radius, c);
}

static PointBatch sample_around(const ConvexPolygon& p, std::size_t count, std::uint64_t seed) {
  return sample_points(count, bounding_box(p.vertices()).scaled(2.0), seed);
}

int main() {
  // --- conversion (test_voronoi.cpp) ---
  {
    const GeneratorSet g = to_voronoi(unit_square());
    CHECK(g.inner == (Point2{0.5, 0.5}));
    CHECK(g.edge_count() == 4);
    CHECK(g.outer[0] == (Point2{0.5, -0.5}));
    CHECK(g.outer[1] == (Point2{1.5, 0.5}));
    CHECK(g.outer[2] == (Point2{0.5, 1.5}));
    CHECK(g.outer[3] == (Point2{-0.5, 0.5}));
    const GeneratorSet t = to_voronoi(validate_polygon({{0, 0}, {1, 0}, {0, 1}}));
    CHECK(std::abs(t.inner.x - 1.0 / 3.0) <= 1e-15 && t.outer[0].x == t.inner.x &&
          t.outer[0].y == -t.inner.y);
    const GeneratorSet p5 = to_voronoi(regular_polygon(5, 1.0));
    for (const Point2& q : p5.outer) CHECK(std::abs(std::hypot(q.x, q.y) - 1.618033988749895) <= 1e-9);
    CHECK(edge_coefficients({0, 0}, {1, 0}) == (EdgeCoefficients{0, 1, 0}));
    CHECK(edge_coefficients({0, 1}, {1, 0}) == (EdgeCoefficients{1, 1, -1}));
    CHECK(thrown_code([] { edge_coefficients({2, 3}, {2, 3}); }) == static_cast<int>(ErrorCode::DegenerateEdge));
    CHECK(reflect_generator({0.5, 0.5}, {0, 1, 0}) == (Point2{0.5, -0.5}));
    CHECK(thrown_code([] { reflect_generator({0.5, 0.5}, {1, 1, -1}); }) ==
          static_cast<int>(ErrorCode::GeneratorCollision));
    const Point2 c = centroid(validate_polygon({{0, 0}, {2, 0}, {2, 1}, {0, 3}}));
    CHECK(std::abs(c.x - 5.0 / 6.0) <= 1e-12 && std::abs(c.y - 13.0 / 12.0) <= 1e-12);
    for (std::uint64_t i = 0; i < 10; ++i) {
      const ConvexPolygon poly = make_test_polygon(i);
      CHECK(to_voronoi(poly) == to_voronoi(poly));  // byte-for-byte reproducible
    }
  }
  // --- validation (test_geometry.cpp) ---
  CHECK(thrown_code([] { validate_polygon({{0, 0}, {1, 0}}); }) == static_cast<int>(ErrorCode::TooFewVertices));
  CHECK(thrown_code([] { validate_polygon({{0, 0}, {1, 0}, {2, 0}, {1, 1}}); }) == static_cast<int>(ErrorCode::NotConvex));
  CHECK(thrown_code([] { validate_polygon({{0, 0}, {1, 0}, {1, 0}, {0, 1}}); }) == static_cast<int>(ErrorCode::DegenerateEdge));
  CHECK(thrown_code([] { validate_polygon({{0, 0}, {1, NAN}, {0, 1}}); }) == static_cast<int>(ErrorCode::NonFinite));
  CHECK(validate_polygon({{0, 0}, {0, 1}, {1, 1}, {1, 0}}).was_reversed());

  // --- engines (test_engines.cpp) ---
  {
    const ConvexPolygon sq = unit_square();
    const GeneratorSet g = to_voronoi(sq);
    CHECK(voronoi_contains(g, {0.5, 0.5}) && !voronoi_contains(g, {2, 2}) && voronoi_contains(g, {1, 0.5}));
    CHECK(ray_crossing_count(sq.vertices(), {0.5, 0.5}) == 1);
    const PointBatch none;
    CHECK(voronoi_contains_batch(g, none).empty());
    CHECK(sign_of_offset_contains_batch(sq, none).empty());
    CHECK(ray_crossing_contains_batch(sq.vertices(), none).empty());
    PointBatch pts;
    pts.push_back({0.5, 0.5});
    pts.push_back({2, 2});
    const InclusionMask expected = {1, 0};
    CHECK(voronoi_contains_batch(g, pts) == expected);
    CHECK(sign_of_offset_contains_batch(sq, pts) == expected);
    CHECK(ray_crossing_contains_batch(sq.vertices(), pts) == expected);
    // closed boundary (acceptance 8)
    PointBatch bnd;
    for (std::size_t k = 0; k < 4; ++k) {
      const Point2 a = sq.vertex(k), b = sq.vertex((k + 1) % 4);
      bnd.push_back(a);
      bnd.push_back(0.5 * (a + b));
    }
    const InclusionMask ones(bnd.size(), 1);
    CHECK(voronoi_contains_batch(g, bnd) == ones);
    CHECK(sign_of_offset_contains_batch(sq, bnd) == ones);
    CHECK(ray_crossing_contains_batch(sq.vertices(), bnd) == ones);
    const PointBatch u = sample_points(10'000, {-1, -1, 2, 2}, 4242);
    CHECK(voronoi_contains_batch(g, u) == sign_of_offset_contains_batch(sq, u));
  }
  {  // concave arrow (test_engines.cpp:73-81)
    const std::vector<Point2> arrow = {{0, 0}, {4, 0}, {4, 4}, {2, 1}, {0, 4}};
    PointBatch pts;
    for (Point2 p : {Point2{2, 2}, Point2{1, 1}, Point2{3, 1}, Point2{-1, 1}}) pts.push_back(p);
    CHECK(ray_crossing_contains_batch(arrow, pts) == (InclusionMask{0, 1, 1, 0}));
  }
  // batch == scalar (acceptance 7) and three-way agreement outside the band (acceptance 1)
  for (std::uint64_t i = 0; i < 8; ++i) {
    const ConvexPolygon poly = make_test_polygon(i);
    const GeneratorSet g = to_voronoi(poly);
    const PointBatch pts = sample_around(poly, 10'000, mix_seed(31, i));
    const InclusionMask mv = voronoi_contains_batch(g, pts);
    const InclusionMask ms = sign_of_offset_contains_batch(poly, pts);
    const InclusionMask mr = ray_crossing_contains_batch(poly.vertices(), pts);
    std::size_t bad = 0;
    for (std::size_t j = 0; j < pts.size(); ++j) {
      bad += mv[j] != voronoi_contains(g, pts.at(j));
      bad += ms[j] != sign_of_offset_contains(poly, pts.at(j));
      bad += mr[j] != ray_crossing_contains(poly.vertices(), pts.at(j));
      if (edge_line_distance(poly, pts.at(j)) > tol::kAgreementBand) bad += (mv[j] != ms[j]) + (mv[j] != mr[j]);
    }
    CHECK(bad == 0);
  }
  {  // work counters (acceptance 5) and thread-count independence
    for (auto [n, m] : {std::pair<std::size_t, std::size_t>{3, 1000}, {15, 10'000}}) {
      const ConvexPolygon poly = regular_polygon(n, 1.0);
      const GeneratorSet g = to_voronoi(poly);
      BatchStats stats;
      const PointBatch pts = sample_around(poly, m, 7);
      const InclusionMask counted = voronoi_contains_batch(g, pts, stats);
      CHECK(stats.distance_evaluations == (n + 1) * m && stats.comparisons == n * m);
      CHECK(counted == voronoi_contains_batch(g, pts, 13));
    }
  }
  {  // concurrent callers on one generator set (test_engines.cpp:243-257)
    const ConvexPolygon poly = make_test_polygon(6);
    const GeneratorSet g = to_voronoi(poly);
    const PointBatch pts = sample_around(poly, 50'000, 555);
    const InclusionMask expected = voronoi_contains_batch(g, pts);
    std::vector<InclusionMask> results(4);
    {
      std::vector<std::jthread> workers;
      for (std::size_t t = 0; t < results.size(); ++t)
        workers.emplace_back([&, t] { results[t] = voronoi_contains_batch(g, pts); });
    }
    for (const InclusionMask& r : results) CHECK(r == expected);
  }
  CHECK(parse_engine("offset") == EngineKind::SignOfOffset && !parse_engine("winding"));
  std::printf("test_vpip_api: %d checks, %d failed\n", g_checks, g_fail);
  return g_fail == 0 ? 0 : 1;
}
