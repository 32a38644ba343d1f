// vpip/error.hpp -- error contract of the vpip API (B200 engine edition).
// Mirrors proj/include/vpip/error.hpp:23-58: the same ErrorCode values in the
// same order (the C-ABI returns them as 1..7) and an Error exception.
#pragma once

#include <stdexcept>
#include <string>
#include <string_view>

namespace vpip {

enum class ErrorCode {
  TooFewVertices,
  NotConvex,
  DegenerateEdge,
  NonFinite,
  GeneratorCollision,
  InvalidParameter,
  ParseError,
};

std::string_view error_code_name(ErrorCode code);

class Error : public std::runtime_error {
 public:
  Error(ErrorCode code, const std::string& message);
  ErrorCode code() const noexcept { return code_; }

 private:
  ErrorCode code_;
};

}  // namespace vpip
