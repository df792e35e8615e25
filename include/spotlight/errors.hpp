// Drop-in for proj/include/spotlight/errors.hpp (the reference's exception
// taxonomy). The C-ABI status codes of include/spl_c.h map 1:1 onto these.
#pragma once

#include <stdexcept>
#include <string>

namespace spotlight {

/// Bad shapes, k outside [1, n], unsupported code lengths (SPL_E_DIMENSION).
struct DimensionError : std::invalid_argument {
    using std::invalid_argument::invalid_argument;
};

/// Malformed on-disk SPLH / SPLC data (SPL_E_FORMAT).
struct FormatError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

/// Non-finite weights or inputs (SPL_E_NUMERIC).
struct NumericError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

/// Ranking-loss error of the reference's trainer (kept for API parity; the
/// GPU decode path never raises it).
struct EmptyPairError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

/// File open / write failures (SPL_E_IO).
struct IoError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

/// CUDA / device failures of the B200 backend (no reference counterpart).
struct DeviceError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

}  // namespace spotlight
