// Dense retrieval instruments on the GPU: the reference's
// oracle_topk (attention_eval.cpp:121-135) — exact float logits q . k_j over
// the causal range, then top_k_indices<float> — and iou (:216-232), the
// retrieval-accuracy metric of the paper's Table 1 (hash top-k vs oracle).
//
// Exactness. causal_logits (attention_eval.cpp:80-91) is the same
// `acc += q[p] * k[p]` loop as attend_subset, and the reference build
// compiles it the same way (oracle/spl_oracle.c ref_dot, pinned against the
// reference library in tests/test_oracle_vs_ref.py): products rounded,
// summed in index order, for the 8-wide and 4-wide vector parts, then
// fused multiply-adds for the < 4 element tail. One thread per key row
// repeats that chain with explicit __fmul_rn / __fadd_rn / __fmaf_rn, so the
// logits — and therefore the indices, ties included — are bit-identical.
//
// Layout: keys [P][cap][d] (f32 or bf16; bf16 widened exactly, i.e. the
// reference fed the same rounded values), q [P][d] f32, logits [P][n_max].
// A warp stages 32 key rows through shared memory with coalesced loads
// (row stride d + 1 floats: the per-lane column reads are conflict-free).
// HBM-bound: n * d * sizeof(K) bytes per problem.
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "spl_launch.cuh"

namespace spl {
namespace {

constexpr int kLgWarps = 4;
constexpr uint32_t kLgMaxD = 256;

template <typename KT>
__device__ __forceinline__ float widen(KT v);
template <>
__device__ __forceinline__ float widen<float>(float v) { return v; }
template <>
__device__ __forceinline__ float widen<__nv_bfloat16>(__nv_bfloat16 v) { return __bfloat162float(v); }

template <typename KT>
__global__ void __launch_bounds__(kLgWarps * 32) k_causal_logits(const float* __restrict__ q,
                                                                 const KT* __restrict__ keys,
                                                                 uint64_t cap, uint32_t d,
                                                                 const uint32_t* n_valid,
                                                                 uint32_t nvalid_div, uint64_t n_max,
                                                                 float scale, float* logits) {
    extern __shared__ float sm[];  // [d] query + [warps][32][d + 1] key rows
    const uint32_t p = blockIdx.y;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    float* sq = sm;
    float* tile = sm + d + (size_t)warp * 32 * (d + 1);
    for (uint32_t i = threadIdx.x; i < d; i += blockDim.x) sq[i] = q[(uint64_t)p * d + i];
    __syncthreads();
    uint64_t nv = n_valid[p / nvalid_div];
    if (nv > n_max) nv = n_max;
    const KT* kp = keys + (uint64_t)p * cap * d;
    const uint32_t n8 = d / 8 * 8, n4 = (d - n8) >= 4 ? n8 + 4 : n8;
    for (uint64_t r0 = ((uint64_t)blockIdx.x * kLgWarps + warp) * 32; r0 < nv;
         r0 += (uint64_t)gridDim.x * kLgWarps * 32) {
        const uint32_t rows = (uint32_t)(nv - r0 < 32 ? nv - r0 : 32);
        for (uint32_t r = 0; r < rows; ++r)
            for (uint32_t c = lane; c < d; c += 32) tile[r * (d + 1) + c] = widen<KT>(kp[(r0 + r) * d + c]);
        __syncwarp();
        if ((uint32_t)lane < rows) {
            const float* kr = tile + lane * (d + 1);
            float acc = 0.0f;
            uint32_t i = 0;
            for (; i < n4; ++i) acc = __fadd_rn(acc, __fmul_rn(sq[i], kr[i]));
            for (; i < d; ++i) acc = __fmaf_rn(sq[i], kr[i], acc);
            logits[(uint64_t)p * n_max + r0 + lane] = __fmul_rn(acc, scale);
        }
        __syncwarp();
    }
}

// iou of two ascending index lists per problem (attention_eval.cpp:216-232):
// |a ∩ b| / |a ∪ b|, 1 when both are empty. Each element of a is looked up
// in b by binary search (both lists strictly ascending).
__global__ void __launch_bounds__(256) k_iou(const uint32_t* a, const uint32_t* cnt_a,
                                             uint64_t a_stride, const uint32_t* b,
                                             const uint32_t* cnt_b, uint64_t b_stride,
                                             double* out) {
    __shared__ uint32_t s_hits;
    const uint32_t p = blockIdx.x;
    const uint32_t na = cnt_a[p], nb = cnt_b[p];
    const uint32_t* ap = a + (uint64_t)p * a_stride;
    const uint32_t* bp = b + (uint64_t)p * b_stride;
    if (threadIdx.x == 0) s_hits = 0;
    __syncthreads();
    uint32_t hits = 0;
    for (uint32_t i = threadIdx.x; i < na; i += blockDim.x) {
        const uint32_t v = ap[i];
        uint32_t lo = 0, hi = nb;
        while (lo < hi) {
            const uint32_t mid = (lo + hi) >> 1;
            if (bp[mid] < v) lo = mid + 1; else hi = mid;
        }
        hits += (lo < nb && bp[lo] == v) ? 1u : 0u;
    }
    for (int o = 16; o > 0; o >>= 1) hits += __shfl_xor_sync(0xffffffffu, hits, o);
    if ((threadIdx.x & 31) == 0 && hits) atomicAdd(&s_hits, hits);
    __syncthreads();
    if (threadIdx.x == 0) {
        const uint64_t uni = (uint64_t)na + nb - s_hits;
        out[p] = uni == 0 ? 1.0 : (double)s_hits / (double)uni;
    }
}

// matmul (matrix.hpp:81-99) as the reference build computes it: every
// output c[i][j] starts at 0 and takes fma(a[i][p], b[p][j], c) for p = 0..k-1
// in order. One thread per output; b (k x n, row-major) is read coalesced.
__global__ void __launch_bounds__(256) k_project(const float* __restrict__ a, uint64_t m,
                                                 uint32_t k, const float* __restrict__ b,
                                                 uint32_t n, float* __restrict__ c) {
    const uint64_t i = blockIdx.y;
    const uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= m || j >= n) return;
    const float* ar = a + i * k;
    float acc = 0.0f;
    for (uint32_t p = 0; p < k; ++p) acc = __fmaf_rn(__ldg(ar + p), __ldg(b + (uint64_t)p * n + j), acc);
    c[i * n + j] = acc;
}

}  // namespace

spl_status project_launch(spl_ctx* ctx, const float* a, uint64_t m, uint32_t k, const float* b,
                          uint32_t n, float* c, cudaStream_t s) {
    if (m == 0 || n == 0) return SPL_OK;
    if (m > 0xFFFFFFFFull / 2) return fail(ctx, SPL_E_DIMENSION, "matmul: too many rows");
    const dim3 grid((n + 255) / 256, (unsigned)m);
    k_project<<<grid, 256, 0, s>>>(a, m, k, b, n, c);
    return after_launch(ctx, "k_project");
}

spl_status causal_logits_launch(spl_ctx* ctx, const float* q, const void* keys, int kv_dtype,
                                uint64_t cap, uint32_t d, uint32_t P, const uint32_t* n_valid,
                                uint32_t nvalid_div, uint64_t n_max, float scale, float* logits,
                                cudaStream_t s) {
    if (d == 0 || d > kLgMaxD)
        return fail(ctx, SPL_E_DIMENSION, "oracle_topk: head dim must be in [1, 256]");
    if (P == 0 || n_max == 0) return SPL_OK;
    const size_t smem = sizeof(float) * (d + (size_t)kLgWarps * 32 * (d + 1));
    const uint64_t tiles = (n_max + kLgWarps * 32 - 1) / (kLgWarps * 32);
    const uint32_t gx = (uint32_t)std::min<uint64_t>(tiles, std::max<uint64_t>(1, (uint64_t)ctx->num_sms * 8 / P + 1));
    const dim3 grid(gx, P);
    const void* fn = kv_dtype == SPL_BF16 ? reinterpret_cast<const void*>(&k_causal_logits<__nv_bfloat16>)
                                          : reinterpret_cast<const void*>(&k_causal_logits<float>);
    SPL_CUDA_TRY(ctx, cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    void* args[] = {const_cast<float**>(&q), const_cast<void**>(&keys), &cap, &d,
                    const_cast<uint32_t**>(&n_valid), &nvalid_div, &n_max, &scale, &logits};
    SPL_CUDA_TRY(ctx, cudaLaunchKernel(fn, grid, dim3(kLgWarps * 32), args, smem, s));
    return after_launch(ctx, "k_causal_logits");
}

spl_status iou_launch(spl_ctx* ctx, const uint32_t* a, const uint32_t* cnt_a, uint64_t a_stride,
                      const uint32_t* b, const uint32_t* cnt_b, uint64_t b_stride, uint32_t P,
                      double* out, cudaStream_t s) {
    if (P == 0) return SPL_OK;
    k_iou<<<P, 256, 0, s>>>(a, cnt_a, a_stride, b, cnt_b, b_stride, out);
    return after_launch(ctx, "k_iou");
}

}  // namespace spl
