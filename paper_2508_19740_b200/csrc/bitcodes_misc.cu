// Device forms of the remaining bitcodes.hpp entry points (sm_100a):
// pack_bits / unpack_bits (bitcodes.cpp:22-57), nxor_scores_into with an
// int32 scores-out buffer (bitcodes.cpp:59-76; the fused K3 path never
// materialises these) and top_k_indices<S> on arbitrary int32/f32/f64
// scores (bitcodes.cpp:89-131) as an exact MSB-first radix select + ordered
// compaction with the reference's tie rule (lower index first).
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

#include "spl_launch.cuh"

namespace spl {

// bitcodes.cpp:22-41: word w of row i = columns {c*W + w}, chunk c at bit 31-c.
__global__ void k_pack_bits(const uint8_t* bits, uint64_t n, uint32_t L, uint32_t* codes) {
    const uint32_t W = L / 32;
    const uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n * W) return;
    const uint64_t i = t / W;
    const uint32_t w = (uint32_t)(t % W);
    const uint8_t* row = bits + i * L;
    uint32_t word = 0;
    for (uint32_t c = 0; c < 32; ++c) word = (word << 1) | (uint32_t)(row[c * W + w] & 1u);
    codes[t] = word;
}

__global__ void k_unpack_bits(const uint32_t* codes, uint64_t n, uint32_t L, uint8_t* bits) {
    const uint32_t W = L / 32;
    const uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n * L) return;
    const uint64_t i = t / L;
    const uint32_t j = (uint32_t)(t % L);
    const uint32_t c = j / W, w = j % W;
    bits[t] = (uint8_t)((codes[i * W + w] >> (31 - c)) & 1u);
}

__global__ void k_nxor_scores(const uint32_t* codes, uint64_t stride_rows, uint32_t W,
                              const uint32_t* qcodes, uint32_t P, const uint32_t* n_valid,
                              uint32_t nvalid_div, uint64_t n_max, int32_t* scores,
                              uint64_t scores_stride, uint32_t* dev_err) {
    const uint32_t p = blockIdx.y;
    uint32_t nv = n_valid[p / nvalid_div];
    if (nv > n_max) {
        if (threadIdx.x == 0 && blockIdx.x == 0) raise_dev_err(dev_err, SPL_DEV_ERR_DIMENSION);
        nv = (uint32_t)n_max;
    }
    const uint32_t* q = qcodes + (uint64_t)p * W;
    const uint32_t* base = codes + (uint64_t)p * stride_rows * W;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nv;
         i += (uint64_t)gridDim.x * blockDim.x) {
        int32_t agree = 0;
        for (uint32_t w = 0; w < W; ++w) agree += __popc(~(__ldg(q + w) ^ __ldg(base + i * W + w)));
        scores[(uint64_t)p * scores_stride + i] = agree;
    }
}

// ---- generic exact top-k (one CTA per score row) -------------------------
// Keys are order-preserving unsigned images of the scores: larger key ==
// ranks ahead. -0.0 is canonicalised to +0.0 (the reference compares with
// != and >, so the two zeros tie).
template <int DT>
__device__ __forceinline__ uint64_t score_key(const void* s, uint64_t i) {
    if constexpr (DT == 0) {
        return (uint64_t)((uint32_t)static_cast<const int32_t*>(s)[i] ^ 0x80000000u);
    } else if constexpr (DT == 1) {
        float f = static_cast<const float*>(s)[i];
        if (f == 0.0f) f = 0.0f;
        const uint32_t u = __float_as_uint(f);
        return (uint64_t)((u & 0x80000000u) ? ~u : (u | 0x80000000u));
    } else {
        double f = static_cast<const double*>(s)[i];
        if (f == 0.0) f = 0.0;
        const uint64_t u = (uint64_t)__double_as_longlong(f);
        return (u & 0x8000000000000000ull) ? ~u : (u | 0x8000000000000000ull);
    }
}

constexpr int kTopkThreads = 1024;

// n_valid (nullable): row p ranks only its first min(n, n_valid[p / div])
// scores and keeps min(k, that) of them (oracle_topk's causal clamp,
// attention_eval.cpp:131); cnt (nullable) receives that count.
template <int DT>
__global__ void __launch_bounds__(kTopkThreads) k_topk_radix(const void* scores, uint64_t n_all,
                                                             uint64_t stride, uint32_t k_all,
                                                             uint32_t* idx, const uint32_t* n_valid,
                                                             uint32_t nvalid_div, uint32_t* cnt) {
    __shared__ uint32_t hist[256];
    __shared__ uint64_t s_prefix, s_mask;
    __shared__ uint32_t s_need;
    __shared__ uint32_t s_warp[kTopkThreads / 32 + 1];
    const uint32_t p = blockIdx.x;
    const uint64_t n = n_valid ? min(n_all, (uint64_t)n_valid[p / nvalid_div]) : n_all;
    const uint32_t k = (uint32_t)min((uint64_t)k_all, n);
    if (cnt && threadIdx.x == 0) cnt[p] = k;
    if (k == 0) return;
    const size_t esz = DT == 0 ? 4 : (DT == 1 ? 4 : 8);
    const void* row = static_cast<const uint8_t*>(scores) + (uint64_t)p * stride * esz;
    const int key_bits = DT == 2 ? 64 : 32;
    if (threadIdx.x == 0) {
        s_prefix = 0;
        s_mask = 0;
        s_need = k;
    }
    __syncthreads();
    for (int shift = key_bits - 8; shift >= 0; shift -= 8) {
        for (int i = threadIdx.x; i < 256; i += kTopkThreads) hist[i] = 0;
        __syncthreads();
        const uint64_t prefix = s_prefix, mask = s_mask;
        for (uint64_t i = threadIdx.x; i < n; i += kTopkThreads) {
            const uint64_t key = score_key<DT>(row, i);
            if ((key & mask) == prefix) atomicAdd(&hist[(key >> shift) & 255u], 1u);
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            uint32_t need = s_need, above = 0;
            int b = 255;
            for (; b > 0; --b) {
                if (above + hist[b] >= need) break;
                above += hist[b];
            }
            s_need = need - above;
            s_prefix = prefix | ((uint64_t)b << shift);
            s_mask = mask | (255ull << shift);
        }
        __syncthreads();
    }
    const uint64_t T = s_prefix;  // key of the k-th best
    const uint32_t take = s_need; // ties (key == T) to keep, lowest index first
    // ordered compaction
    uint32_t carry_sel = 0, carry_eq = 0;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (uint64_t base = 0; base < n; base += kTopkThreads) {
        const uint64_t i = base + threadIdx.x;
        uint64_t key = 0;
        bool gt = false, eq = false;
        if (i < n) {
            key = score_key<DT>(row, i);
            gt = key > T;
            eq = key == T;
        }
        // eq rank (exclusive) within the tile
        const uint32_t eq_ball = __ballot_sync(0xffffffffu, eq);
        if (lane == 0) s_warp[warp] = __popc(eq_ball);
        __syncthreads();
        uint32_t eq_before_warp = 0, eq_tile = 0;
        for (int w = 0; w < kTopkThreads / 32; ++w) {
            if (w < warp) eq_before_warp += s_warp[w];
            eq_tile += s_warp[w];
        }
        const uint32_t eq_rank = carry_eq + eq_before_warp + __popc(eq_ball & ((1u << lane) - 1u));
        const bool sel = gt || (eq && eq_rank < take);
        __syncthreads();
        const uint32_t sel_ball = __ballot_sync(0xffffffffu, sel);
        if (lane == 0) s_warp[warp] = __popc(sel_ball);
        __syncthreads();
        uint32_t sel_before_warp = 0, sel_tile = 0;
        for (int w = 0; w < kTopkThreads / 32; ++w) {
            if (w < warp) sel_before_warp += s_warp[w];
            sel_tile += s_warp[w];
        }
        if (sel)
            idx[(uint64_t)p * k_all + carry_sel + sel_before_warp +
                __popc(sel_ball & ((1u << lane) - 1u))] = (uint32_t)i;
        carry_sel += sel_tile;
        carry_eq += eq_tile;
        __syncthreads();
    }
}

spl_status pack_bits_launch(spl_ctx* ctx, const uint8_t* bits, uint64_t n, uint32_t L,
                            uint32_t* codes, cudaStream_t s) {
    const uint64_t work = n * (L / 32);
    if (work == 0) return SPL_OK;
    k_pack_bits<<<(unsigned)((work + 255) / 256), 256, 0, s>>>(bits, n, L, codes);
    return after_launch(ctx, "k_pack_bits");
}

spl_status unpack_bits_launch(spl_ctx* ctx, const uint32_t* codes, uint64_t n, uint32_t L,
                              uint8_t* bits, cudaStream_t s) {
    const uint64_t work = n * L;
    if (work == 0) return SPL_OK;
    k_unpack_bits<<<(unsigned)((work + 255) / 256), 256, 0, s>>>(codes, n, L, bits);
    return after_launch(ctx, "k_unpack_bits");
}

spl_status nxor_scores_launch(spl_ctx* ctx, const uint32_t* codes, uint64_t stride_rows,
                              uint32_t L, const uint32_t* qcodes, uint32_t P,
                              const uint32_t* n_valid, uint32_t nvalid_div, uint64_t n_max,
                              int32_t* scores, uint64_t scores_stride, cudaStream_t s) {
    if (P == 0 || n_max == 0) return SPL_OK;
    const uint64_t blocks = (n_max + 255) / 256;
    dim3 grid((unsigned)(blocks < 4096 ? blocks : 4096), P);
    k_nxor_scores<<<grid, 256, 0, s>>>(codes, stride_rows, L / 32, qcodes, P, n_valid, nvalid_div,
                                       n_max, scores, scores_stride, ctx->dev_err);
    return after_launch(ctx, "k_nxor_scores");
}

spl_status top_k_launch(spl_ctx* ctx, const void* scores, int dtype, uint32_t P, uint64_t n,
                        uint64_t stride, uint32_t k, uint32_t* idx, cudaStream_t s,
                        const uint32_t* n_valid, uint32_t nvalid_div, uint32_t* cnt) {
    if (P == 0) return SPL_OK;
    switch (dtype) {
        case 0: k_topk_radix<0><<<P, kTopkThreads, 0, s>>>(scores, n, stride, k, idx, n_valid, nvalid_div, cnt); break;
        case 1: k_topk_radix<1><<<P, kTopkThreads, 0, s>>>(scores, n, stride, k, idx, n_valid, nvalid_div, cnt); break;
        case 2: k_topk_radix<2><<<P, kTopkThreads, 0, s>>>(scores, n, stride, k, idx, n_valid, nvalid_div, cnt); break;
        default: return fail(ctx, SPL_E_DIMENSION, "top_k_indices: unknown score dtype");
    }
    return after_launch(ctx, "k_topk_radix");
}

}  // namespace spl
