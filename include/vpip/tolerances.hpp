// vpip/tolerances.hpp -- numeric thresholds (values of
// proj/include/vpip/tolerances.hpp:20-42).
#pragma once

namespace vpip::tol {

inline constexpr double kConvexityCross = 1e-12;      // collinear / reflex vertex
inline constexpr double kDegenerateEdgeSq = 1e-24;    // zero-length edge
inline constexpr double kGeneratorCollision = 1e-12;  // centroid on an edge line
inline constexpr double kGeneratorResidual = 1e-9;    // mirror-invariant residuals
inline constexpr double kAgreementBand = 1e-9;        // engine cross-check band

}  // namespace vpip::tol
