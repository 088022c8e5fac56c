// tloom/errors.hpp -- exception taxonomy of the tensorloom API (B200 build).
//
// Same hierarchy as the reference (proj/include/tloom/errors.hpp:9-31) so that callers' catch
// clauses and CHECK_THROWS_AS assertions keep working:
//   Error <- ShapeError <- BoundsError,   Error <- FormatError <- ValueError.
// The C ABI (tloom_b200.h) reports these as TLB_ERR_* codes; tloom::detail::raise() maps them back.
#pragma once

#include <stdexcept>
#include <string>

namespace tloom {

struct Error : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct ShapeError : Error {
  using Error::Error;
};
struct BoundsError : ShapeError {
  using ShapeError::ShapeError;
};
struct FormatError : Error {
  using Error::Error;
};
struct ValueError : FormatError {
  using FormatError::FormatError;
};

namespace detail {
// Throws the exception type matching a C-ABI status code (no-op for TLB_OK).
void raise(int status);
}  // namespace detail

}  // namespace tloom
