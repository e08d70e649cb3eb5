// rlplan vocabulary shared by every module.
//
// Drop-in for /root/reference/proj/include/rlplan/common.hpp:9-32 — same
// namespace, type aliases, helpers and exception type, so that callers of
// the reference planner compile unchanged against this library.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

namespace rlplan {

// Scalar aliases (reference common.hpp:11-15). A DeviceId is the global
// index node * gpus_per_node + gpu.
using Count = std::int64_t;
using Bytes = std::int64_t;
using Seconds = double;
using NodeId = int;
using DeviceId = int;

// reference common.hpp:17
inline bool is_power_of_two(Count v) { return v > 0 && (v & (v - 1)) == 0; }

// reference common.hpp:19 (positive operands)
inline Count ceil_div(Count num, Count den) { return (num + den - 1) / den; }

// Raised whenever an input breaks a documented invariant (reference
// common.hpp:21-25). It is-a std::invalid_argument so generic handlers work.
class ValidationError : public std::invalid_argument {
 public:
  explicit ValidationError(const std::string& message) : std::invalid_argument(message) {}
};

// Non-throwing validator result (reference common.hpp:27-30).
struct Violation {
  std::string message;
};

// --- additions used by the realloc module (not in the reference header) ---

inline Count gcd_count(Count a, Count b) {
  while (b != 0) {
    const Count t = a % b;
    a = b;
    b = t;
  }
  return a;
}

inline Count lcm_count(Count a, Count b) { return a / gcd_count(a, b) * b; }

}  // namespace rlplan
