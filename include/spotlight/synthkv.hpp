// Drop-in for the dump half of proj/include/spotlight/synthkv.hpp
// (synthkv.hpp:36-47): the SPLQ query/key dump the trainer reads
// (`spotlight train --dump`). The synthetic cone sampler (ConeSpec,
// sample_cone) is data generation, not part of the B200 path, and is not
// provided.
#pragma once

#include <string>

#include "spotlight/matrix.hpp"

namespace spotlight {

// In-memory form of a query/key dump.
struct QkDump {
    Matrix<float> queries;
    Matrix<float> keys;
};

// Dump file, magic "SPLQ": u32 version=1, u32 n_queries, u32 n_keys, u32 d,
// then the query block and key block, row-major little-endian f32.
// write_dump: DimensionError on differing widths, NumericError on non-finite
// values; read_dump: FormatError on a bad magic / version / truncation /
// non-finite payload (the reference's messages).
void write_dump(const std::string& path, const Matrix<float>& queries, const Matrix<float>& keys);
QkDump read_dump(const std::string& path);

}  // namespace spotlight
