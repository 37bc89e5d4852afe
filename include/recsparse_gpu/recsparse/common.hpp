// recsparse_gpu -- the reference's C++ API (proj/include/recsparse/*.hpp) on
// the B200 build: same namespace, types, signatures and exceptions, so code
// written against the reference (its own unit suites included) relinks
// unchanged against librecsparse_gpu.so, which calls the C-ABI of rsgpu.h.
//
// common.hpp: the exception taxonomy of common.hpp:24-39.  C-ABI status codes
// map back 1:1 (RS_ERR_CONFIG -> ConfigError, RS_ERR_INVARIANT ->
// InvariantError, RS_ERR_IO -> IoError, RS_ERR_RANGE -> std::out_of_range,
// RS_ERR_CUDA / RS_ERR_CAPACITY -> std::runtime_error).
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>

namespace recsparse {

class ConfigError : public std::runtime_error {
 public:
  explicit ConfigError(const std::string& what) : std::runtime_error(what) {}
};
class IoError : public std::runtime_error {
 public:
  explicit IoError(const std::string& what) : std::runtime_error(what) {}
};
class InvariantError : public std::runtime_error {
 public:
  explicit InvariantError(const std::string& what) : std::runtime_error(what) {}
};

constexpr bool is_power_of_two(uint64_t x) { return x && (x & (x - 1)) == 0; }

namespace gpu {
// Throws the exception of a non-zero rsgpu status (message from rs_last_error).
void check(int status, const char* what);
}  // namespace gpu

}  // namespace recsparse
