// Test-only header (not part of the drop-in): the reference's test sources
// include spotlight/synthkv.hpp for its synthetic cone sampler (ConeSpec,
// sample_cone — data generation, out of scope for the B200 path). This header
// is the drop-in's synthkv.hpp plus those declarations (synthkv.hpp:11-35 of
// the reference); oracle/Makefile's `reftests` target compiles the
// reference's own src/synthkv.cpp against it as a test-data generator, with
// its dump functions renamed so the drop-in's write_dump/read_dump stay the
// ones under test.
#pragma once

#include <cstdint>
#include <vector>

#include "../../../../include/spotlight/synthkv.hpp"

namespace spotlight {

struct ConeSpec {
    std::uint32_t dim = 128;
    std::vector<double> query_axis;
    std::vector<double> key_axis;
    double angular_spread = 0.3;
    double axis_cos = 0.0;
    double norm_mean = 0.0;
    double norm_std = 0.0;
    double outlier_prob = 0.0;
    double outlier_scale = 4.0;
    std::uint64_t seed = 0;

    double resolved_norm_mean() const;
    double resolved_norm_std() const;
    void validate() const;
};

enum class ConeSide { query, key };

Matrix<float> sample_cone(const ConeSpec& spec, std::uint32_t count, ConeSide side);

}  // namespace spotlight
