// vpip/sampling.hpp -- seeded workload generators (API of
// proj/include/vpip/sampling.hpp:27-45, same semantics: std::mt19937_64,
// top-53-bit uniforms, splitmix64 seed mixing).
#pragma once

#include <cstdint>

#include "vpip/engines.hpp"
#include "vpip/geometry.hpp"

namespace vpip {

ConvexPolygon regular_polygon(std::size_t n, double circumradius, Point2 center = {});
ConvexPolygon random_convex_polygon(std::size_t n, std::uint64_t seed,
                                    double circumradius = 1.0, Point2 center = {});
PointBatch sample_points(std::size_t count, const Box& box, std::uint64_t seed);
std::uint64_t mix_seed(std::uint64_t seed, std::uint64_t salt);

}  // namespace vpip
