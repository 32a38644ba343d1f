// vpip/voronoi.hpp -- polygon -> Voronoi generator conversion.
// API of proj/include/vpip/voronoi.hpp:25-73. to_voronoi runs on the B200
// (prep kernel, paper_2007_15385_b200/csrc/prep.cu).
#pragma once

#include <cstddef>
#include <vector>

#include "vpip/geometry.hpp"

namespace vpip {

struct EdgeCoefficients {
  double a = 0.0;
  double b = 0.0;
  double c = 0.0;
  friend constexpr bool operator==(const EdgeCoefficients&, const EdgeCoefficients&) = default;
};

EdgeCoefficients edge_coefficients(Point2 q_i, Point2 q_j,
                                   double degenerate_sq = tol::kDegenerateEdgeSq);
double line_distance(const EdgeCoefficients& e, Point2 p);
Point2 foot_of_perpendicular(Point2 p0, const EdgeCoefficients& e);
Point2 reflect_generator(Point2 p0, const EdgeCoefficients& e,
                         double collision_rel = tol::kGeneratorCollision);

struct GeneratorSet {
  Point2 inner;
  std::vector<Point2> outer;  // outer[k] mirrors inner across edge k (v[k] -> v[k+1])
  std::size_t edge_count() const noexcept { return outer.size(); }
  friend bool operator==(const GeneratorSet&, const GeneratorSet&) = default;
};

GeneratorSet to_voronoi(const ConvexPolygon& polygon);
double edge_line_distance(const ConvexPolygon& polygon, Point2 p);

}  // namespace vpip
