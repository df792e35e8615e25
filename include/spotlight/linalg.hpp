// Drop-in for proj/include/spotlight/linalg.hpp (linalg.hpp:9-22): the
// host-side f64 helpers behind the reference's rotation-based initialisers
// (qr_rotation_init, downproj_init). Initialisation only — not on the decode
// path — so they run on the host, with the reference's exact rounding
// sequence (every multiply-add its Release build contracts is an explicit
// fma), bit-identical to it (tests/cpp/test_host_pins.cpp vs oracle/_ref).
#pragma once

#include <cstdint>

#include "spotlight/matrix.hpp"

namespace spotlight {

/// Orthogonal factor Q of a Householder QR of a square matrix (dense).
/// DimensionError if a is not square.
Matrix<double> qr_orthogonal_factor(const Matrix<double>& a);

/// Determinant by LU with partial pivoting. DimensionError if not square.
double lu_determinant(Matrix<double> a);

/// Q of the QR of an i.i.d. N(0, 1) d x d draw from
/// mt19937_64(derive_seed(seed, attempt)); first column negated when det < 0,
/// so the result is in SO(d). DimensionError for d < 1.
Matrix<double> random_rotation(std::uint32_t d, std::uint64_t seed);

}  // namespace spotlight
