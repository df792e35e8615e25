// Generic dense helpers behind the reference's templated host API
// (matrix.hpp:81-99 `matmul<T>`; hashers.hpp:70-98 the double instantiations
// of mlp_forward / linear_hash / mlp_hash, soft_sign, soft_codes,
// downproj_scores). Not on the decode hot path — the drop-in composes these
// for callers of those generic entry points, so that every compute call of
// the drop-in stays a GPU launch.
//
// Rounding follows the reference build (Release, -march=native contracts
// `c += a * b` into one fused multiply-add): matmul output c[i][j] starts at
// 0 and takes fma(a[i][p], b[p][j], c) for p = 0..k-1 in order — bit-exact
// for f32 and f64. The f32 SiLU uses the glibc expf port (spl_expf.cuh,
// bit-exact); the f64 SiLU uses CUDA's exp (<= 1 ulp from glibc's), which the
// reference's double-precision tests bound at 1e-12 relative.
// Compiled with -fmad=false (Makefile EXACT_FLAGS): every rounding explicit.
#include <cuda_runtime.h>
#include <stdint.h>

#include "spl_expf.cuh"
#include "spl_internal.cuh"

namespace spl {
namespace {

__device__ __forceinline__ float fma_t(float a, float b, float c) { return __fmaf_rn(a, b, c); }
__device__ __forceinline__ double fma_t(double a, double b, double c) { return __fma_rn(a, b, c); }

template <typename T>
__global__ void __launch_bounds__(256) k_matmul(const T* __restrict__ a, uint64_t m, uint64_t k,
                                                const T* __restrict__ b, uint64_t n,
                                                T* __restrict__ c) {
    const uint64_t i = blockIdx.y;
    const uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= m || j >= n) return;
    const T* ar = a + i * k;
    T acc = T(0);
    for (uint64_t p = 0; p < k; ++p) acc = fma_t(__ldg(ar + p), __ldg(b + p * n + j), acc);
    c[i * n + j] = acc;
}

__device__ __forceinline__ float silu_t(float y) {
    return __fdiv_rn(y, __fadd_rn(1.0f, spl_expf(-y)));
}
__device__ __forceinline__ double silu_t(double y) { return __ddiv_rn(y, __dadd_rn(1.0, exp(-y))); }
__device__ __forceinline__ float add_t(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ double add_t(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ float mul_t(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ double mul_t(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ float div_t(float a, float b) { return __fdiv_rn(a, b); }
__device__ __forceinline__ double div_t(double a, double b) { return __ddiv_rn(a, b); }

// op 0 SPL_MAP_BIAS_SILU: silu(x[i][j] + bias[j]) (hashers.cpp:97-100)
// op 1 SPL_MAP_SOFT_SIGN: gamma x / (1 + gamma |x|) (hashers.hpp:150-153;
//      the build contracts the denominator: fma(gamma, |x|, 1))
// op 2 SPL_MAP_SIGN_BITS: byte (x >= 0), sign(0) -> 1 (hashers.cpp:19-28)
template <typename T>
__global__ void __launch_bounds__(256) k_map(const T* __restrict__ x, uint64_t rows, uint64_t cols,
                                             const T* __restrict__ bias, T gamma, int op,
                                             void* __restrict__ out) {
    const uint64_t total = rows * cols;
    for (uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total;
         t += (uint64_t)gridDim.x * blockDim.x) {
        const T v = x[t];
        if (op == SPL_MAP_BIAS_SILU) {
            static_cast<T*>(out)[t] = silu_t(add_t(v, bias[t % cols]));
        } else if (op == SPL_MAP_SOFT_SIGN) {
            const T den = fma_t(gamma, v < T(0) ? -v : v, T(1));
            static_cast<T*>(out)[t] = div_t(mul_t(gamma, v), den);
        } else {
            static_cast<uint8_t*>(out)[t] = v >= T(0) ? 1u : 0u;
        }
    }
}

}  // namespace
}  // namespace spl

using namespace spl;

namespace {
inline cudaStream_t S(void* s) { return static_cast<cudaStream_t>(s); }
bool real_dtype(int dt) { return dt == SPL_F32 || dt == SPL_F64; }
}  // namespace

spl_status spl_matmul(spl_ctx* ctx, int dtype, const void* a, uint64_t m, uint64_t k, const void* b,
                      uint64_t n, void* c, void* stream) {
    if (!ctx) return SPL_E_STATE;
    if (!real_dtype(dtype)) return fail(ctx, SPL_E_DIMENSION, "matmul: dtype must be f32 or f64");
    if (m == 0 || n == 0) return SPL_OK;
    if (!a || !b || !c) return fail(ctx, SPL_E_STATE, "matmul: null device pointer");
    if (m > 65535ull * 1024 || n > (1ull << 31))
        return fail(ctx, SPL_E_DIMENSION, "matmul: output too large for the generic kernel");
    if (k == 0) {
        SPL_CUDA_TRY(ctx, cudaMemsetAsync(c, 0, m * n * (dtype == SPL_F64 ? 8 : 4), S(stream)));
        return SPL_OK;
    }
    // rows beyond the grid's y limit are taken in chunks
    for (uint64_t r0 = 0; r0 < m; r0 += 65535) {
        const uint64_t mr = m - r0 < 65535 ? m - r0 : 65535;
        const dim3 grid((unsigned)((n + 255) / 256), (unsigned)mr);
        if (dtype == SPL_F64)
            k_matmul<double><<<grid, 256, 0, S(stream)>>>(static_cast<const double*>(a) + r0 * k, mr, k,
                                                          static_cast<const double*>(b), n,
                                                          static_cast<double*>(c) + r0 * n);
        else
            k_matmul<float><<<grid, 256, 0, S(stream)>>>(static_cast<const float*>(a) + r0 * k, mr, k,
                                                         static_cast<const float*>(b), n,
                                                         static_cast<float*>(c) + r0 * n);
        spl_status st = after_launch(ctx, "k_matmul");
        if (st) return st;
    }
    return SPL_OK;
}

spl_status spl_map(spl_ctx* ctx, int dtype, int op, const void* x, uint64_t rows, uint64_t cols,
                   const void* bias, double gamma, void* out, void* stream) {
    if (!ctx) return SPL_E_STATE;
    if (!real_dtype(dtype)) return fail(ctx, SPL_E_DIMENSION, "map: dtype must be f32 or f64");
    if (op < SPL_MAP_BIAS_SILU || op > SPL_MAP_SIGN_BITS) return fail(ctx, SPL_E_DIMENSION, "map: unknown op");
    if (rows == 0 || cols == 0) return SPL_OK;
    if (!x || !out || (op == SPL_MAP_BIAS_SILU && !bias))
        return fail(ctx, SPL_E_STATE, "map: null device pointer");
    if (op == SPL_MAP_SOFT_SIGN && !(gamma > 0.0))
        return fail(ctx, SPL_E_DIMENSION, "soft_sign: gamma must be positive");
    const uint64_t total = rows * cols;
    const unsigned blocks = (unsigned)(total / 256 + 1 < 4096 ? total / 256 + 1 : 4096);
    if (dtype == SPL_F64)
        k_map<double><<<blocks, 256, 0, S(stream)>>>(static_cast<const double*>(x), rows, cols,
                                                     static_cast<const double*>(bias), gamma, op, out);
    else
        k_map<float><<<blocks, 256, 0, S(stream)>>>(static_cast<const float*>(x), rows, cols,
                                                    static_cast<const float*>(bias), (float)gamma, op, out);
    return after_launch(ctx, "k_map");
}
