// Bit-exact expf for the exact-mode encoder (K1).
//
// The reference's SiLU (hashers.cpp:30-33, `z / (1 + std::exp(-z))`) calls
// glibc's expf. On an x86-64 host with FMA+AVX2, glibc 2.39 dispatches (ifunc)
// to its FMA build of sysdeps/ieee754/flt-32/e_expf.c. This is that algorithm
// restated with every contraction GCC made in that build written as an
// explicit fma (read from the shipped libm.so.6 disassembly: __expf_fma at
// 0x7dc40), and the table/constants read from its .rodata. Pure IEEE double
// arithmetic, so host (g++ -ffp-contract=off) and device (__fma_rn/__dmul_rn)
// evaluate identically; tools/check_expf_exhaustive.cpp compares it with
// libm's expf over all 2^32 inputs (0 mismatches), and the GPU parity tests
// check K1's pre-activations bitwise against the reference.
// Origin / licence: the algorithm, its 32-entry table and constants are
// glibc's (sysdeps/ieee754/flt-32/e_expf.c, contributed by Arm from
// optimized-routines; LGPL-2.1+ in glibc, MIT / Apache-2.0 WITH LLVM-exception
// in Arm optimized-routines). This is a restatement for bit parity, not a copy
// of the reference repository.
#pragma once
#include <stdint.h>
#include <string.h>

#if defined(__CUDACC__)
#define SPL_HD __host__ __device__ __forceinline__
#else
#include <math.h>
#define SPL_HD static inline
#endif

namespace spl_expf_detail {

// 2^(i/32) tabulated as uint64 bit patterns minus (i << 47) (EXP2F_TABLE_BITS=5).
#define SPL_EXPF_TAB { \
    0x3ff0000000000000ull, 0x3fefd9b0d3158574ull, 0x3fefb5586cf9890full, 0x3fef9301d0125b51ull, \
    0x3fef72b83c7d517bull, 0x3fef54873168b9aaull, 0x3fef387a6e756238ull, 0x3fef1e9df51fdee1ull, \
    0x3fef06fe0a31b715ull, 0x3feef1a7373aa9cbull, 0x3feedea64c123422ull, 0x3feece086061892dull, \
    0x3feebfdad5362a27ull, 0x3feeb42b569d4f82ull, 0x3feeab07dd485429ull, 0x3feea47eb03a5585ull, \
    0x3feea09e667f3bcdull, 0x3fee9f75e8ec5f74ull, 0x3feea11473eb0187ull, 0x3feea589994cce13ull, \
    0x3feeace5422aa0dbull, 0x3feeb737b0cdc5e5ull, 0x3feec49182a3f090ull, 0x3feed503b23e255dull, \
    0x3feee89f995ad3adull, 0x3feeff76f2fb5e47ull, 0x3fef199bdd85529cull, 0x3fef3720dcef9069ull, \
    0x3fef5818dcfba487ull, 0x3fef7c97337b9b5full, 0x3fefa4afa2a490daull, 0x3fefd0765b6e4540ull}
#if defined(__CUDACC__)
__device__ __constant__ uint64_t kTabDev[32] = SPL_EXPF_TAB;
#endif
static const uint64_t kTabHost[32] = SPL_EXPF_TAB;

SPL_HD uint64_t tab(uint32_t i) {
#if defined(__CUDA_ARCH__)
    return kTabDev[i];
#else
    return kTabHost[i];
#endif
}

SPL_HD double fma_rn(double a, double b, double c) {
#if defined(__CUDA_ARCH__)
    return __fma_rn(a, b, c);
#else
    return fma(a, b, c);
#endif
}
SPL_HD double mul_rn(double a, double b) {
#if defined(__CUDA_ARCH__)
    return __dmul_rn(a, b);
#else
    return a * b;
#endif
}
SPL_HD double sub_rn(double a, double b) {
#if defined(__CUDA_ARCH__)
    return __dsub_rn(a, b);
#else
    return a - b;
#endif
}
SPL_HD uint32_t f2u(float f) {
    uint32_t u;
    memcpy(&u, &f, 4);
    return u;
}
SPL_HD float u2f(uint32_t u) {
    float f;
    memcpy(&f, &u, 4);
    return f;
}
SPL_HD uint64_t d2u(double d) {
    uint64_t u;
    memcpy(&u, &d, 8);
    return u;
}
SPL_HD double u2d(uint64_t u) {
    double d;
    memcpy(&d, &u, 8);
    return d;
}

}  // namespace spl_expf_detail

SPL_HD float spl_expf(float x) {
    using namespace spl_expf_detail;
    const double kShift = 0x1.8p+52;
    const double kInvLn2N = 0x1.71547652b82fep+5;  // 32 / ln 2
    const double kC0 = 0x1.c6af84b912394p-20;
    const double kC1 = 0x1.ebfce50fac4f3p-13;
    const double kC2 = 0x1.62e42ff0c52d6p-6;
    const uint32_t ix = f2u(x);
    const uint32_t abstop = (ix >> 20) & 0x7ffu;
    if (abstop >= 0x42bu) {  // |x| >= 88 or nan
        if (ix == 0xff800000u) return 0.0f;                  // -inf
        if (abstop >= 0x7f8u) return x + x;                  // inf / nan
        if (x > 0x1.62e42ep6f) return u2f(0x7f800000u);      // __math_oflowf
        if (x < -0x1.9fe368p6f) return 0.0f;                 // __math_uflowf
        if (x < -0x1.9d1d9ep6f) return u2f(0x00000001u);     // __math_may_uflowf: 0x1p-149
    }
    const double xd = (double)x;
    double kd = fma_rn(kInvLn2N, xd, kShift);  // contracted z + SHIFT
    const uint64_t ki = d2u(kd);
    kd = sub_rn(kd, kShift);
    const double r = fma_rn(kInvLn2N, xd, -kd);  // contracted z - kd
    const uint64_t t = tab((uint32_t)(ki & 31u)) + (ki << 47);
    const double s = u2d(t);
    const double z = fma_rn(r, kC0, kC1);
    const double r2 = mul_rn(r, r);
    double y = fma_rn(r, kC2, 1.0);
    y = fma_rn(z, r2, y);
    y = mul_rn(y, s);
#if defined(__CUDA_ARCH__)
    return __double2float_rn(y);
#else
    return (float)y;
#endif
}
