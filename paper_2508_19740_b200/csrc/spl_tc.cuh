// Operand layout of the tcgen05 bulk encoder (K2, encode_tc.cu), shared with
// the host-side weight preparation in capi.cu.
//
// Every UMMA operand is K-major bf16 with K = 128, stored as two 64-element
// K blocks; block kb is `rows` rows of 128 bytes, 128-byte swizzled: the
// 16-byte chunk c of row r sits at chunk position c ^ (r % 8) (the canonical
// SWIZZLE_128B K-major layout, 8-row atoms of 1024 B, atoms 1024 B apart).
// The shared-memory descriptor of k-step s (16 elements = 32 B) starts at
// block (s / 4) + 32 B * (s % 4); the hardware applies the XOR from the
// address bits, so every block must be 1024-byte aligned.
#pragma once
#include <stdint.h>

namespace spl {

constexpr uint32_t kTcK = 128;       // contraction length of both GEMMs (d = h = 128)
constexpr uint32_t kTcTileM = 128;   // keys per tile (UMMA M)

// byte offset of element (r, k) in an operand of `rows` rows
__host__ __device__ __forceinline__ uint32_t tc_sw_off(uint32_t r, uint32_t k, uint32_t rows) {
    const uint32_t kb = k >> 6, kk = k & 63u;
    return kb * rows * 128u + r * 128u + ((((kk >> 3) ^ (r & 7u)) & 7u) << 4) + ((kk & 7u) << 1);
}

// bytes of one operand (rows x 128 bf16)
__host__ __device__ __forceinline__ uint32_t tc_operand_bytes(uint32_t rows) { return rows * 256u; }

// host: f32 -> bf16 bits, round to nearest even (finite inputs)
inline uint16_t tc_bf16_bits(float f) {
    uint32_t u;
    __builtin_memcpy(&u, &f, 4);
    u += 0x7FFFu + ((u >> 16) & 1u);
    return (uint16_t)(u >> 16);
}

}  // namespace spl
