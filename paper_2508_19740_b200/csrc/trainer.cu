// Hasher training on the GPU: the reference's train_hasher
// (trainer.cpp:520-645) for the MLP and linear coders with the pairwise
// ranking loss (ranking_loss.cpp:80-145 sampling, trainer.cpp:297-380 soft
// loss), AdamW (trainer.cpp:100-143), global-norm clipping (:83-97), the
// warmup + cosine schedule (:35-46) and the holdout IoU (:472-518).
//
// Division of labour. The host keeps what is sequential and tiny: the
// mt19937_64 draws (sequence pick, partition seed, randperm prefixes — the
// same std:: engine and distributions as the reference, so the sampled
// (query, top, other) sets are identical), the schedule, and pow(beta, t)
// for the bias corrections. Everything that touches a matrix is a kernel:
// exact q.k logits, the per-row descending order (bitonic sort in shared
// memory), soft-code forward passes over every key, the ranking loss and its
// gradient, backward through the coder, clipping, AdamW, and the holdout
// retrieval (K1 codes -> K3 top-k vs float top-k of the logits -> IoU).
//
// Arithmetic follows the reference build's evaluation order per output
// (compiled with EXACT_FLAGS; every rounding is an explicit intrinsic):
//  * matmul / add_matmul_at (matrix.hpp:81-99, :121-138): one fused
//    multiply-add chain per output, in index order, starting from the
//    output's current value;
//  * matmul_bt (matrix.hpp:101-117): rounded products summed in index order
//    for the vectorised part, fused tail (as attention_eval's dot, see
//    dense_retrieval.cu);
//  * double dots of float soft codes (trainer.cpp:313-335): products are
//    exact in double, so only the (sequential) add order matters;
//  * per-key soft-code gradients: the reference adds g * sq to a key row
//    query by query; here dk[key] is one fma chain over the selected queries
//    in order, reading a dense [key][query] matrix of the g values — the same
//    sequence of roundings.
// Two reductions differ in order from the reference's sequential loops (the
// reported loss sum and the clipping norm's sum of squares); both are
// deterministic here and agree to a few ulps of a double. Double exp/log1p
// are CUDA's (<= 1-2 ulp from glibc's): the pair gradients are rounded to
// float before use, so they match unless a double lands within an ulp of a
// float rounding boundary. tests/test_gpu_trainer.py checks weights, records
// and holdout IoU against the unmodified reference's train_hasher.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cmath>
#include <cstdlib>
#include <numeric>
#include <random>
#include <string>
#include <vector>

#include "spl_expf.cuh"
#include "spl_launch.cuh"

namespace spl {
namespace {

constexpr uint32_t kMaxSortKeys = 16384;  // order sort chunk (shared memory); longer rows merge

// halt codes (device): the reference throws out of train_loop at that point
enum : uint32_t { HALT_NONE = 0, HALT_EMPTY = 1, HALT_NONFINITE = 2 };

struct TrainDev {
    uint32_t halt;          // HALT_*
    uint32_t halt_iter;
    uint32_t step;          // AdamW step (applied updates)
    uint32_t skipped;       // non-finite gradient steps
    uint32_t skip_now;      // this iteration's gradients are non-finite
    float scale;            // this iteration's clipping factor
    double bc1, bc2;        // this iteration's bias corrections
    double loss_acc, viol_acc;
    unsigned long long pairs;  // valid pairs of the current (iteration, batch) element
};

// ------------------------------------------------------------ scalar pieces
__device__ __forceinline__ float sigmoid_f(float z) {
    return __fdiv_rn(1.0f, __fadd_rn(1.0f, spl_expf(-z)));
}
// trainer.cpp:181-185 (silu_grad): s * (1 + z * (1 - s)), z*(1-s)+1 fused
__device__ __forceinline__ float silu_grad_f(float z) {
    const float s = sigmoid_f(z);
    return __fmul_rn(s, __fmaf_rn(z, __fsub_rn(1.0f, s), 1.0f));
}
// hashers.hpp:151-159: gamma*z / (1 + gamma*|z|), gamma / (1 + gamma*|z|)^2
__device__ __forceinline__ float soft_sign_f(float z, float g) {
    return __fdiv_rn(__fmul_rn(g, z), __fmaf_rn(g, fabsf(z), 1.0f));
}
__device__ __forceinline__ float soft_sign_grad_f(float z, float g) {
    const float den = __fmaf_rn(g, fabsf(z), 1.0f);
    return __fdiv_rn(g, __fmul_rn(den, den));
}
// trainer.cpp:295-297
__device__ __forceinline__ double softplus_d(double x) {
    return x > 0.0 ? __dadd_rn(x, log1p(exp(-x))) : log1p(exp(x));
}
// the pair gradient of trainer.cpp:349-351 (beta * (1 - sigmoid(logit)) * inv)
__device__ __forceinline__ double pair_g(double logit, double beta, double inv) {
    const double sg = __ddiv_rn(1.0, __dadd_rn(1.0, exp(-logit)));
    return __dmul_rn(__dmul_rn(beta, __dsub_rn(1.0, sg)), inv);
}
__device__ __forceinline__ uint32_t n4_of(uint32_t k) {
    const uint32_t n8 = k / 8 * 8;
    return (k - n8) >= 4 ? n8 + 4 : n8;
}

// ------------------------------------------------------------ exact logits
// logits[i][j] = matmul_bt(Q, K)[i][j] * scale (trainer.cpp:394-400), all
// q x n entries. 64 x 64 output tile per block, 4 x 4 per thread; the chain
// of each output walks p in order across the 32-wide shared-memory chunks.
__global__ void __launch_bounds__(256) k_logits(const float* __restrict__ Q, const float* __restrict__ K,
                                                uint32_t q, uint32_t n, uint32_t d, float scale,
                                                float* __restrict__ out) {
    __shared__ float qs[64][33], ks[64][33];
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    const uint32_t r0 = blockIdx.y * 64, c0 = blockIdx.x * 64;
    const uint32_t n4 = n4_of(d);
    float acc[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = 0.0f;
    for (uint32_t p0 = 0; p0 < d; p0 += 32) {
        const uint32_t w = min(32u, d - p0);
        for (uint32_t e = threadIdx.x; e < 64 * 32; e += 256) {
            const uint32_t r = e / 32, c = e % 32;
            qs[r][c] = (r0 + r < q && c < w) ? Q[(uint64_t)(r0 + r) * d + p0 + c] : 0.0f;
            ks[r][c] = (c0 + r < n && c < w) ? K[(uint64_t)(c0 + r) * d + p0 + c] : 0.0f;
        }
        __syncthreads();
        for (uint32_t pp = 0; pp < w; ++pp) {
            const bool fused = p0 + pp >= n4;
            float a[4], b[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) a[i] = qs[ty + 16 * i][pp];
#pragma unroll
            for (int j = 0; j < 4; ++j) b[j] = ks[tx + 16 * j][pp];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j)
                    acc[i][j] = fused ? __fmaf_rn(a[i], b[j], acc[i][j])
                                      : __fadd_rn(acc[i][j], __fmul_rn(a[i], b[j]));
        }
        __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const uint32_t r = r0 + ty + 16 * i, c = c0 + tx + 16 * j;
            if (r < q && c < n) out[(uint64_t)r * n + c] = __fmul_rn(acc[i][j], scale);
        }
}

// ------------------------------------------------------------ order
// build_topk_order (ranking_loss.cpp:30-59) for one row per block: causally
// valid keys by descending score, ties to the lower index, masked keys last
// in index order. Keys (~orderable(score) << 32 | j) sorted ascending by a
// bitonic network over the next power of two (pads sort last); -0 == +0.
__device__ __forceinline__ uint32_t orderable(float f) {
    uint32_t u = __float_as_uint(f);
    if (u == 0x80000000u) u = 0u;
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
// One C-key chunk (C a power of two <= kMaxSortKeys) of a row per block:
// rows longer than C are sorted chunk by chunk here and merged below. Pads
// (j >= n) sort last and stay unique: (0xFFFFFFFF << 32) | j.
__global__ void __launch_bounds__(1024) k_order(const float* __restrict__ logits, uint32_t n,
                                                uint32_t C, uint32_t row0,
                                                uint32_t* __restrict__ order,
                                                unsigned long long* __restrict__ runs) {
    extern __shared__ unsigned long long keys[];
    const uint32_t row = row0 + blockIdx.y, c0 = blockIdx.x * C;
    const uint32_t valid = min(row + 1, n);
    const float* s = logits + (uint64_t)row * n;
    for (uint32_t t = threadIdx.x; t < C; t += blockDim.x) {
        const uint32_t j = c0 + t;
        uint32_t hi = 0xFFFFFFFFu;
        if (j < valid) hi = ~orderable(s[j]);
        keys[t] = ((unsigned long long)hi << 32) | j;
    }
    __syncthreads();
    for (uint32_t k = 2; k <= C; k <<= 1)
        for (uint32_t j = k >> 1; j > 0; j >>= 1) {
            for (uint32_t i = threadIdx.x; i < C; i += blockDim.x) {
                const uint32_t l = i ^ j;
                if (l > i) {
                    const unsigned long long a = keys[i], b = keys[l];
                    const bool up = (i & k) == 0;
                    if ((a > b) == up) {
                        keys[i] = b;
                        keys[l] = a;
                    }
                }
            }
            __syncthreads();
        }
    if (gridDim.x == 1) {  // the whole row fits one chunk
        for (uint32_t j = threadIdx.x; j < n; j += blockDim.x)
            order[(uint64_t)row * n + j] = (uint32_t)keys[j];
    } else {
        const uint64_t rowlen = (uint64_t)gridDim.x * C;
        for (uint32_t t = threadIdx.x; t < C; t += blockDim.x)
            runs[(uint64_t)blockIdx.y * rowlen + c0 + t] = keys[t];
    }
}

// One merge pass over sorted runs of length R (keys unique): each key's
// output position = its rank in its own run + its rank in the partner run.
__global__ void k_order_merge(const unsigned long long* __restrict__ src,
                              unsigned long long* __restrict__ dst, uint64_t rowlen, uint64_t R,
                              uint64_t total) {
    for (uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
         e += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t y = e / rowlen, i = e % rowlen;
        const unsigned long long* row = src + y * rowlen;
        const unsigned long long key = row[i];
        const uint64_t r = i / R, pb = (r ^ 1) * R;
        uint64_t pos = i;
        if (pb < rowlen) {
            const uint64_t plen = min(R, rowlen - pb);
            uint64_t lo = 0, hi = plen;  // count of partner keys < key
            while (lo < hi) {
                const uint64_t mid = (lo + hi) >> 1;
                if (row[pb + mid] < key) lo = mid + 1; else hi = mid;
            }
            pos = (r & ~1ull) * R + (i - r * R) + lo;
        }
        dst[y * rowlen + pos] = key;
    }
}

__global__ void k_order_extract(const unsigned long long* __restrict__ src, uint64_t rowlen,
                                uint32_t n, uint32_t row0, uint32_t rows,
                                uint32_t* __restrict__ order) {
    const uint64_t total = (uint64_t)rows * n;
    for (uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
         e += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t y = e / n, j = e % n;
        order[(row0 + y) * (uint64_t)n + j] = (uint32_t)src[y * rowlen + j];
    }
}

// ------------------------------------------------------------ forward
// MlpCoder / LinearCoder / DownProjCoder forward (trainer.cpp:199-217,
// :245-250, :275-277) over m rows (rows[] selects rows of x when given):
// MLP z1 = x W1 (+ b1), a1 = z1 * sigmoid(z1), z2 = a1 W2; linear z2 = x P;
// soft = soft_sign(z2) (downproj: soft = x P). 16 rows per block; each
// thread owns output columns, one fma chain per (row, column).
constexpr int kFwdRows = 16;     // rows per block
constexpr int kFwdThreads = 256; // 128 column lanes x 2 row groups of 8
constexpr int kFwdRg = kFwdRows / (kFwdThreads / 128);
// one layer for this thread's row group: acc[r] = FMA chain over p of
// in[r][p] * W[p][j] (matrix.hpp:81-99). W in shared memory (staged once per
// block by cp.async) or, for shapes too large for it, read through L1/L2
// 32 weights ahead.
template <bool WSMEM>
__device__ __forceinline__ void fwd_layer(const float* in, uint32_t K, const float* W,
                                          uint32_t ncol, uint32_t j, float (&acc)[kFwdRg]) {
#pragma unroll
    for (int r = 0; r < kFwdRg; ++r) acc[r] = 0.0f;
    uint32_t p = 0;
    if constexpr (WSMEM) {
        for (; p < K; ++p) {
            const float w = W[(size_t)p * ncol + j];
#pragma unroll
            for (int r = 0; r < kFwdRg; ++r) acc[r] = __fmaf_rn(in[r * K + p], w, acc[r]);
        }
        return;
    } else {
    for (; p + 32 <= K; p += 32) {
        float w[32];
#pragma unroll
        for (int u = 0; u < 32; ++u) w[u] = __ldg(W + (uint64_t)(p + u) * ncol + j);
#pragma unroll
        for (int u = 0; u < 32; ++u)
#pragma unroll
            for (int r = 0; r < kFwdRg; ++r) acc[r] = __fmaf_rn(in[r * K + p + u], w[u], acc[r]);
    }
    for (; p < K; ++p) {
        const float w = W[(uint64_t)p * ncol + j];
#pragma unroll
        for (int r = 0; r < kFwdRg; ++r) acc[r] = __fmaf_rn(in[r * K + p], w, acc[r]);
    }
    }
}

// n floats global -> shared, 16-byte copies when both sides allow it
__device__ __forceinline__ void cp_async_f32(float* dst, const float* src, uint64_t n) {
    const uint32_t ds = (uint32_t)__cvta_generic_to_shared(dst);
    if ((n & 3u) == 0 && (ds & 15u) == 0 && (reinterpret_cast<uintptr_t>(src) & 15u) == 0) {
        for (uint64_t e = 4 * (uint64_t)threadIdx.x; e < n; e += 4 * (uint64_t)blockDim.x)
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(ds + (uint32_t)e * 4),
                         "l"(src + e)
                         : "memory");
    } else {
        for (uint64_t e = threadIdx.x; e < n; e += blockDim.x)
            asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(ds + (uint32_t)e * 4),
                         "l"(src + e)
                         : "memory");
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
}

template <int KIND, bool WSMEM>  // KIND: SPL_HASHER_MLP / SPL_HASHER_LINEAR / 2 = downproj
__global__ void __launch_bounds__(kFwdThreads) k_forward(const float* __restrict__ x, const uint32_t* rows,
                                                         uint32_t m, uint32_t d, uint32_t h, uint32_t L,
                                                         const float* __restrict__ w1,
                                                         const float* __restrict__ b1,
                                                         const float* __restrict__ w2, float gamma,
                                                         float* z1, float* a1, float* z2, float* soft,
                                                         const TrainDev* st, float* xcopy) {
    if (st->halt) return;
    extern __shared__ float sm[];
    float* xs = sm;                       // [kFwdRows][d]
    float* as = sm + kFwdRows * d;        // [kFwdRows][h] (MLP)
    float* w1s = as + (KIND == SPL_HASHER_MLP ? kFwdRows * h : 0);  // [d][h | L]
    float* w2s = w1s;  // MLP: layer-2 weights reuse the layer-1 buffer (2 blocks / SM)
    const uint32_t r0 = blockIdx.x * kFwdRows;
    const uint32_t nr = min((uint32_t)kFwdRows, m - r0);
    for (uint32_t r = 0; r < kFwdRows; ++r) {  // async row staging, zero rows past m
        const bool ok = r < nr;
        const float* src = ok ? x + (uint64_t)(rows ? rows[r0 + r] : r0 + r) * d : x;
        for (uint32_t c = threadIdx.x; c < d; c += blockDim.x)
            asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(
                             (uint32_t)__cvta_generic_to_shared(xs + r * d + c)),
                         "l"(ok ? src + c : x), "r"(ok ? 4 : 0)
                         : "memory");
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
    if (WSMEM) {  // group 2: layer-1 weights (layer 2's are staged after layer 1)
        cp_async_f32(w1s, w1, (uint64_t)d * (KIND == SPL_HASHER_MLP ? h : L));
        asm volatile("cp.async.wait_group 0;" ::: "memory");
    } else {
        asm volatile("cp.async.wait_group 0;" ::: "memory");
    }
    __syncthreads();
    if (xcopy)  // the gathered query rows, kept for the weight gradients (gather_rows)
        for (uint32_t e = threadIdx.x; e < nr * d; e += blockDim.x) xcopy[(uint64_t)r0 * d + e] = xs[e];
    const uint32_t lane = threadIdx.x & 127, rg = threadIdx.x >> 7;
    const uint32_t rbase = rg * kFwdRg;  // this thread's rows: rbase .. rbase + kFwdRg - 1
    const float* in = xs + rbase * d;
    uint32_t K = d;
    const float* W = WSMEM ? w1s : w1;
    float acc[kFwdRg];
    if (KIND == SPL_HASHER_MLP) {
        for (uint32_t j = lane; j < h; j += 128) {
            fwd_layer<WSMEM>(in, d, W, h, j, acc);
            const float bj = b1[j];
#pragma unroll
            for (int r = 0; r < kFwdRg; ++r) {
                const uint32_t rr = rbase + r;
                const float z = __fadd_rn(acc[r], bj);
                const float a = __fmul_rn(z, sigmoid_f(z));
                as[rr * h + j] = a;
                if (rr < nr) {
                    z1[(uint64_t)(r0 + rr) * h + j] = z;
                    a1[(uint64_t)(r0 + rr) * h + j] = a;
                }
            }
        }
        __syncthreads();  // layer 1 done with the weight buffer
        if (WSMEM) {
            cp_async_f32(w2s, w2, (uint64_t)h * L);
            asm volatile("cp.async.wait_group 0;" ::: "memory");
            __syncthreads();
        }
        in = as + rbase * h;
        K = h;
        W = WSMEM ? w2s : w2;
    }
    for (uint32_t j = lane; j < L; j += 128) {
        fwd_layer<WSMEM>(in, K, W, L, j, acc);
#pragma unroll
        for (int r = 0; r < kFwdRg; ++r) {
            const uint32_t rr = rbase + r;
            if (rr < nr) {
                const uint64_t o = (uint64_t)(r0 + rr) * L + j;
                if (KIND != 2) z2[o] = acc[r];
                soft[o] = KIND == 2 ? acc[r] : soft_sign_f(acc[r], gamma);
            }
        }
    }
}

// ------------------------------------------------------------ partition
// partition_topk's index gather (ranking_loss.cpp:118-141): key =
// order[row][pos]; an entry is valid iff key < the row's causal offset.
// Adds this (iteration, element)'s valid pair count (sum over rows of
// valid_top * valid_oth) into st->pairs.
__global__ void __launch_bounds__(256) k_partition(const uint32_t* __restrict__ order, uint32_t n,
                                                   uint32_t k_full, const uint32_t* qrows,
                                                   const uint32_t* top_pos, uint32_t T,
                                                   const uint32_t* oth_pos, uint32_t O,
                                                   uint32_t* top_idx, uint32_t* oth_idx,
                                                   TrainDev* st) {
    if (st->halt) return;
    __shared__ uint32_t s_t[8], s_o[8];
    const uint32_t qi = blockIdx.x;
    const uint32_t row = qrows[qi];
    const uint32_t valid = min(row + 1, n);
    const uint32_t* ro = order + (uint64_t)row * n;
    uint32_t ct = 0, co = 0;
    for (uint32_t i = threadIdx.x; i < T; i += blockDim.x) {
        const uint32_t key = ro[top_pos[i]];
        const bool ok = key < valid;
        top_idx[(uint64_t)qi * T + i] = ok ? key : ~0u;
        ct += ok;
    }
    for (uint32_t j = threadIdx.x; j < O; j += blockDim.x) {
        const uint32_t key = ro[k_full + oth_pos[j]];
        const bool ok = key < valid;
        oth_idx[(uint64_t)qi * O + j] = ok ? key : ~0u;
        co += ok;
    }
    for (int o = 16; o; o >>= 1) {
        ct += __shfl_xor_sync(~0u, ct, o);
        co += __shfl_xor_sync(~0u, co, o);
    }
    if ((threadIdx.x & 31) == 0) {
        s_t[threadIdx.x >> 5] = ct;
        s_o[threadIdx.x >> 5] = co;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t a = 0, b = 0;
        for (uint32_t w = 0; w < blockDim.x / 32; ++w) {
            a += s_t[w];
            b += s_o[w];
        }
        atomicAdd(&st->pairs, (unsigned long long)a * b);
    }
}

// ------------------------------------------------------------ ranking loss
// ranking_soft_loss (trainer.cpp:299-380), three kernels:
//  k_rank_dots   B_i = <sq, sk_top_i>, C_j = <sq, sk_oth_j> in double, one
//                thread per entry (products of floats are exact in double:
//                only the sequential add order matters);
//  k_rank_pairs  one thread per (i, j) pair: softplus(-(beta (B_i - C_j) -
//                alpha)), the violation flag and the pair gradient g, stored
//                as gp[qi][i][j] (invalid pairs: 0); loss / violation partial
//                per block;
//  k_rank_grad   gb[i] = -sum_j g (j ascending), gc[j] = sum_i g (i
//                ascending) — the reference's accumulation orders — then dq
//                = one fma chain over the non-zero entries (top first, then
//                other), and the g values of the touched keys into G[key][qi]
//                for the key-side chain.
__global__ void __launch_bounds__(128) k_rank_dots(const float* __restrict__ softq,
                                                   const float* __restrict__ softk, uint32_t L,
                                                   const uint32_t* top_idx, uint32_t T,
                                                   const uint32_t* oth_idx, uint32_t O,
                                                   double* bc, TrainDev* st, uint32_t iter) {
    if (st->halt) return;
    if (st->pairs == 0) {  // EmptyPairError (trainer.cpp:303-305)
        if (blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) {
            st->halt = HALT_EMPTY;
            st->halt_iter = iter;
        }
        return;
    }
    extern __shared__ float sq[];  // [L]
    const uint32_t qi = blockIdx.x;
    for (uint32_t p = threadIdx.x; p < L; p += blockDim.x) sq[p] = softq[(uint64_t)qi * L + p];
    __syncthreads();
    const uint32_t e = blockIdx.y * blockDim.x + threadIdx.x;
    if (e >= T + O) return;
    const uint32_t key = e < T ? top_idx[(uint64_t)qi * T + e] : oth_idx[(uint64_t)qi * O + e - T];
    double acc = 0.0;
    if (key != ~0u) {
        const float* sk = softk + (uint64_t)key * L;
        uint32_t p = 0;
        for (; p + 8 <= L; p += 8) {
            float v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) v[u] = __ldg(sk + p + u);
#pragma unroll
            for (int u = 0; u < 8; ++u) acc = __dadd_rn(acc, __dmul_rn((double)sq[p + u], (double)v[u]));
        }
        for (; p < L; ++p) acc = __dadd_rn(acc, __dmul_rn((double)sq[p], (double)sk[p]));
    }
    bc[(uint64_t)qi * (T + O) + e] = acc;
}

constexpr int kPairThreads = 256;
constexpr int kPairsPerThread = 4;
__global__ void __launch_bounds__(kPairThreads) k_rank_pairs(const double* __restrict__ bc,
                                                             const uint32_t* top_idx, uint32_t T,
                                                             const uint32_t* oth_idx, uint32_t O,
                                                             double beta, double alpha,
                                                             double* __restrict__ gp,
                                                             double* loss_part,
                                                             unsigned long long* viol_part,
                                                             const TrainDev* st) {
    if (st->halt) return;
    __shared__ double s_loss[kPairThreads / 32];
    __shared__ unsigned long long s_viol[kPairThreads / 32];
    const uint32_t qi = blockIdx.x;
    const double inv = __ddiv_rn(1.0, (double)st->pairs);
    double loss = 0.0;
    unsigned long long viol = 0;
    // kPairsPerThread pairs per thread (block-strided): fewer loss partials
    for (int u = 0; u < kPairsPerThread; ++u) {
        const uint64_t e = ((uint64_t)blockIdx.y * kPairsPerThread + u) * kPairThreads + threadIdx.x;
        if (e >= (uint64_t)T * O) break;
        const uint32_t i = (uint32_t)(e / O), j = (uint32_t)(e % O);
        double g = 0.0;
        if (top_idx[(uint64_t)qi * T + i] != ~0u && oth_idx[(uint64_t)qi * O + j] != ~0u) {
            const double* row = bc + (uint64_t)qi * (T + O);
            const double z = __dsub_rn(row[i], row[T + j]);
            const double logit = __fma_rn(beta, z, -alpha);
            loss = __dadd_rn(loss, softplus_d(-logit));
            viol += z < 0.0;
            g = pair_g(logit, beta, inv);
        }
        gp[(uint64_t)qi * T * O + e] = g;
    }
    for (int o = 16; o; o >>= 1) {
        loss = __dadd_rn(loss, __shfl_xor_sync(~0u, loss, o));
        viol += __shfl_xor_sync(~0u, viol, o);
    }
    if ((threadIdx.x & 31) == 0) {
        s_loss[threadIdx.x >> 5] = loss;
        s_viol[threadIdx.x >> 5] = viol;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double a = 0.0;
        unsigned long long v = 0;
        for (int w = 0; w < kPairThreads / 32; ++w) {
            a = __dadd_rn(a, s_loss[w]);
            v += s_viol[w];
        }
        loss_part[(uint64_t)qi * gridDim.y + blockIdx.y] = a;
        viol_part[(uint64_t)qi * gridDim.y + blockIdx.y] = v;
    }
}

__global__ void __launch_bounds__(256) k_rank_grad(const float* __restrict__ softk, uint32_t L,
                                                   const uint32_t* top_idx, uint32_t T,
                                                   const uint32_t* oth_idx, uint32_t O,
                                                   uint32_t Qs, const double* __restrict__ gp,
                                                   float* G, float* dsq, const TrainDev* st) {
    if (st->halt) return;
    extern __shared__ double dsm[];
    double* gsum = dsm;  // [T + O]: gb then gc
    const uint32_t qi = blockIdx.x;
    const uint32_t* ti = top_idx + (uint64_t)qi * T;
    const uint32_t* oi = oth_idx + (uint64_t)qi * O;
    const double* g = gp + (uint64_t)qi * T * O;
    // invalid pairs hold g = +0: acc - 0 and acc + 0 leave acc unchanged
    // (acc starts at +0 and the pair gradients are >= 0), so the chains run
    // over every slot. gb: 32-column tiles of g staged through shared memory
    // (coalesced), each thread continuing its row's chain across tiles.
    // gb: each thread walks its row of g in order, 32 loads in flight ahead of
    // the chain (rows are contiguous; L1 serves the rest of each sector)
    for (uint32_t i = threadIdx.x; i < T; i += blockDim.x) {
        const double* row = g + (uint64_t)i * O;
        double acc = 0.0;
        uint32_t j = 0;
        for (; j + 32 <= O; j += 32) {
            double v[32];
#pragma unroll
            for (int u = 0; u < 32; ++u) v[u] = row[j + u];
#pragma unroll
            for (int u = 0; u < 32; ++u) acc = __dsub_rn(acc, v[u]);
        }
        for (; j < O; ++j) acc = __dsub_rn(acc, row[j]);
        gsum[i] = acc;
    }
    for (uint32_t i = threadIdx.x; i < T; i += blockDim.x)
        if (ti[i] == ~0u) gsum[i] = 0.0;
    for (uint32_t j = threadIdx.x; j < O; j += blockDim.x) {
        double acc = 0.0;
        if (oi[j] != ~0u) {
            uint32_t i = 0;
            for (; i + 8 <= T; i += 8) {
                double v[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) v[u] = g[(uint64_t)(i + u) * O + j];
#pragma unroll
                for (int u = 0; u < 8; ++u) acc = __dadd_rn(acc, v[u]);
            }
            for (; i < T; ++i) acc = __dadd_rn(acc, g[(uint64_t)i * O + j]);
        }
        gsum[T + j] = acc;
    }
    __syncthreads();
    // compact the non-zero entries (top first, then other, each in order):
    // per-warp ballots, one running offset per 256-entry round
    float* eg = reinterpret_cast<float*>(gsum + T + O);   // [T + O]
    uint32_t* ek = reinterpret_cast<uint32_t*>(eg + T + O);  // [T + O]
    __shared__ uint32_t s_ne, s_wc[8];
    if (threadIdx.x == 0) s_ne = 0;
    __syncthreads();
    const uint32_t lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    for (uint32_t e0 = 0; e0 < T + O; e0 += blockDim.x) {
        const uint32_t e = e0 + threadIdx.x;
        const double v = e < T + O ? gsum[e] : 0.0;
        const bool nz = v != 0.0;
        const uint32_t bal = __ballot_sync(~0u, nz);
        if (lane == 0) s_wc[wid] = __popc(bal);
        __syncthreads();
        uint32_t base = s_ne;
        for (uint32_t w = 0; w < wid; ++w) base += s_wc[w];
        if (nz) {
            const uint32_t pos = base + __popc(bal & ((1u << lane) - 1u));
            eg[pos] = __double2float_rn(v);
            ek[pos] = e < T ? ti[e] : oi[e - T];
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            uint32_t t = 0;
            for (uint32_t w = 0; w < blockDim.x / 32; ++w) t += s_wc[w];
            s_ne += t;
        }
        __syncthreads();
    }
    const uint32_t ne = s_ne;
    for (uint32_t p = threadIdx.x; p < L; p += blockDim.x) {
        float dq = 0.0f;
        uint32_t e = 0;
        for (; e + 32 <= ne; e += 32) {  // 32 row loads in flight ahead of the chain
            float v[32];
#pragma unroll
            for (int u = 0; u < 32; ++u) v[u] = __ldg(softk + (uint64_t)ek[e + u] * L + p);
#pragma unroll
            for (int u = 0; u < 32; ++u) dq = __fmaf_rn(eg[e + u], v[u], dq);
        }
        for (; e < ne; ++e) dq = __fmaf_rn(eg[e], softk[(uint64_t)ek[e] * L + p], dq);
        dsq[(uint64_t)qi * L + p] = dq;
    }
    for (uint32_t e = threadIdx.x; e < ne; e += blockDim.x) G[(uint64_t)ek[e] * Qs + qi] = eg[e];
}

// ------------------------------------------------------------ reconstruction loss
// recon_soft_loss (trainer.cpp:383-419): draft = matmul_bt(soft_q, soft_k)
// (rounded products in order, fused tail), diff = draft - true logit over
// the causal range, loss = sum diff^2 / count, g = float(2 / count * diff);
// d soft_q = matmul(g, soft_k) (one fma chain over the keys), d soft_k +=
// g^T soft_q (k_dsoft_keys over G[key][qi] = g[qi][key]).
__global__ void __launch_bounds__(256) k_recon(const float* __restrict__ softq,
                                               const float* __restrict__ softk, uint32_t L,
                                               const float* __restrict__ logits, uint32_t n,
                                               const uint32_t* qrows, uint32_t Qs, double scale,
                                               float* G, double* loss_part, const TrainDev* st) {
    if (st->halt) return;
    extern __shared__ float sq[];  // [L]
    __shared__ double s_l[8];
    const uint32_t qi = blockIdx.x;
    const uint32_t row = qrows[qi];
    const uint32_t valid = min(row + 1, n);
    for (uint32_t p = threadIdx.x; p < L; p += blockDim.x) sq[p] = softq[(uint64_t)qi * L + p];
    __syncthreads();
    const uint32_t n4 = n4_of(L);
    double loss = 0.0;
    for (uint32_t j = blockIdx.y * blockDim.x + threadIdx.x; j < valid; j += gridDim.y * blockDim.x) {
        const float* sk = softk + (uint64_t)j * L;
        float acc = 0.0f;
        uint32_t p = 0;
        for (; p < n4; ++p) acc = __fadd_rn(acc, __fmul_rn(sq[p], __ldg(sk + p)));
        for (; p < L; ++p) acc = __fmaf_rn(sq[p], __ldg(sk + p), acc);
        const double diff = __dsub_rn((double)acc, (double)logits[(uint64_t)row * n + j]);
        loss = __fma_rn(diff, diff, loss);
        G[(uint64_t)j * Qs + qi] = __double2float_rn(__dmul_rn(scale, diff));
    }
    for (int o = 16; o; o >>= 1) loss = __dadd_rn(loss, __shfl_xor_sync(~0u, loss, o));
    if ((threadIdx.x & 31) == 0) s_l[threadIdx.x >> 5] = loss;
    __syncthreads();
    if (threadIdx.x == 0) {
        double a = 0.0;
        for (int w = 0; w < 8; ++w) a = __dadd_rn(a, s_l[w]);
        loss_part[(uint64_t)qi * gridDim.y + blockIdx.y] = a;
    }
}

__global__ void __launch_bounds__(128) k_recon_dq(const float* __restrict__ G,
                                                  const float* __restrict__ softk, uint32_t L,
                                                  uint32_t n, const uint32_t* qrows, uint32_t Qs,
                                                  float invb, float* __restrict__ dsq,
                                                  const TrainDev* st) {
    if (st->halt) return;
    const uint32_t qi = blockIdx.x;
    const uint32_t valid = min(qrows[qi] + 1, n);
    for (uint32_t p = threadIdx.x; p < L; p += blockDim.x) {
        float dq = 0.0f;
        uint32_t j = 0;
        for (; j + 16 <= valid; j += 16) {
            float gv[16], kv[16];
#pragma unroll
            for (int u = 0; u < 16; ++u) {
                gv[u] = G[(uint64_t)(j + u) * Qs + qi];
                kv[u] = __ldg(softk + (uint64_t)(j + u) * L + p);
            }
#pragma unroll
            for (int u = 0; u < 16; ++u)
                if (gv[u] != 0.0f) dq = __fmaf_rn(gv[u], kv[u], dq);
        }
        for (; j < valid; ++j) {
            const float g = G[(uint64_t)j * Qs + qi];
            if (g != 0.0f) dq = __fmaf_rn(g, softk[(uint64_t)j * L + p], dq);
        }
        dsq[(uint64_t)qi * L + p] = invb != 1.0f ? __fmul_rn(dq, invb) : dq;
    }
}

// loss = sum of the query partials * inv_pairs; non-finite -> NumericError
// (trainer.cpp:587-590); accumulates the iteration record over the batch.
__global__ void k_loss_finalize(const double* loss_part, const unsigned long long* viol_part,
                                uint32_t nparts, uint32_t b, uint32_t batch, uint32_t iter,
                                double* rec, TrainDev* st, double recon_count) {
    if (st->halt) return;
    __shared__ double s_l[256];
    __shared__ unsigned long long s_v[256];
    const double inv = st->pairs ? __ddiv_rn(1.0, (double)st->pairs) : 0.0;
    double a = 0.0;
    unsigned long long c = 0;
    uint32_t q = threadIdx.x;
    for (; q + 7 * blockDim.x < nparts; q += 8 * blockDim.x) {  // fixed order per thread
        double lv[8];
        unsigned long long vv[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            lv[u] = loss_part[q + u * blockDim.x];
            vv[u] = viol_part[q + u * blockDim.x];
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            a = __dadd_rn(a, lv[u]);
            c += vv[u];
        }
    }
    for (; q < nparts; q += blockDim.x) {
        a = __dadd_rn(a, loss_part[q]);
        c += viol_part[q];
    }
    s_l[threadIdx.x] = a;
    s_v[threadIdx.x] = c;
    __syncthreads();
    for (uint32_t o = blockDim.x / 2; o; o >>= 1) {
        if (threadIdx.x < o) {
            s_l[threadIdx.x] = __dadd_rn(s_l[threadIdx.x], s_l[threadIdx.x + o]);
            s_v[threadIdx.x] += s_v[threadIdx.x + o];
        }
        __syncthreads();
    }
    if (threadIdx.x) return;
    const double s = s_l[0];
    const unsigned long long v = s_v[0];
    // ranking: sums x (1 / valid pairs) (trainer.cpp:377-379); reconstruction:
    // MSE = sum / count, no violation rate (trainer.cpp:383-419, :571-586)
    const double loss = recon_count > 0.0 ? __ddiv_rn(s, recon_count) : __dmul_rn(s, inv);
    const double vr = recon_count > 0.0 ? 0.0 : __dmul_rn((double)v, inv);
    if (!isfinite(loss)) {
        st->halt = HALT_NONFINITE;
        st->halt_iter = iter;
        return;
    }
    st->loss_acc = b == 0 ? loss : __dadd_rn(st->loss_acc, loss);
    st->viol_acc = b == 0 ? vr : __dadd_rn(st->viol_acc, vr);
    if (b + 1 == batch) {
        rec[3 * (uint64_t)iter] = __ddiv_rn(st->loss_acc, (double)batch);
        rec[3 * (uint64_t)iter + 1] = __ddiv_rn(st->viol_acc, (double)batch);
    }
    st->pairs = 0;  // the next element's count starts from zero
}

// d soft_k = G^T-chain: dk[key][p] = fma over the selected queries in order
// of G[key][qi] * sq[qi][p] (zero G entries are the reference's skipped
// pairs); x (1/batch) when batch > 1 (trainer.cpp:591-595).
// large query sets (no query_subsample): one thread per (key, code position)
__global__ void __launch_bounds__(256) k_dsoft_keys_flat(const float* __restrict__ G,
                                                         const float* __restrict__ softq, uint32_t Qs,
                                                         uint32_t n, uint32_t L, float invb,
                                                         float* __restrict__ dsk, const TrainDev* st) {
    if (st->halt) return;
    const uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= (uint64_t)n * L) return;
    const uint64_t key = e / L;
    const uint32_t p = (uint32_t)(e % L);
    float acc = 0.0f;
    for (uint32_t q = 0; q < Qs; ++q) {
        const float g = G[key * Qs + q];
        if (g != 0.0f) acc = __fmaf_rn(g, softq[(uint64_t)q * L + p], acc);
    }
    dsk[e] = invb != 1.0f ? __fmul_rn(acc, invb) : acc;
}

// softq and this block's G rows staged in shared memory; each thread runs the
// chains of 8 keys for one code position
constexpr int kDkKeys = 16;  // keys per block (2 groups of 8 per 128-column lane set)
__global__ void __launch_bounds__(256) k_dsoft_keys(const float* __restrict__ G,
                                                    const float* __restrict__ softq, uint32_t Qs,
                                                    uint32_t n, uint32_t L, float invb,
                                                    float* __restrict__ dsk, const TrainDev* st) {
    if (st->halt) return;
    extern __shared__ float dk_sm[];
    float* sq = dk_sm;                        // [Qs][L] soft query codes
    float* gs = dk_sm + (size_t)Qs * L;       // [kDkKeys][Qs] g values of this block's keys
    const uint32_t key0 = blockIdx.x * kDkKeys;
    const uint32_t nk = min((uint32_t)kDkKeys, n - key0);
    cp_async_f32(sq, softq, (uint64_t)Qs * L);
    for (uint32_t e = threadIdx.x; e < kDkKeys * Qs; e += blockDim.x)
        gs[e] = e < nk * Qs ? G[(uint64_t)key0 * Qs + e] : 0.0f;
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    __syncthreads();
    const uint32_t kg = (threadIdx.x >> 7) * (kDkKeys / 2);  // this thread's 8 keys
    for (uint32_t p = threadIdx.x & 127; p < L; p += 128) {
        float acc[kDkKeys / 2];
#pragma unroll
        for (int k = 0; k < kDkKeys / 2; ++k) acc[k] = 0.0f;
        for (uint32_t q = 0; q < Qs; ++q) {  // one fma chain per key, queries in order
            const float sv = sq[(size_t)q * L + p];
#pragma unroll
            for (int k = 0; k < kDkKeys / 2; ++k) {
                const float g = gs[(kg + k) * Qs + q];
                if (g != 0.0f) acc[k] = __fmaf_rn(g, sv, acc[k]);
            }
        }
#pragma unroll
        for (int k = 0; k < kDkKeys / 2; ++k)
            if (kg + k < nk)
                dsk[(uint64_t)(key0 + kg + k) * L + p] = invb != 1.0f ? __fmul_rn(acc[k], invb) : acc[k];
    }
}

__global__ void k_transpose(const float* __restrict__ a, uint32_t rows, uint32_t cols,
                            float* __restrict__ at) {  // at[c][r] = a[r][c]
    for (uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; e < (uint64_t)rows * cols;
         e += (uint64_t)gridDim.x * blockDim.x)
        at[(e % cols) * rows + e / cols] = a[e];
}

__global__ void k_scale(float* x, uint64_t n, float s, const TrainDev* st) {
    if (st->halt) return;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x)
        x[i] = __fmul_rn(x[i], s);
}

// ------------------------------------------------------------ backward
// dz = d_soft * soft_sign_grad(z) (trainer.cpp:222-225, :253-257)
__global__ void k_dz(const float* __restrict__ dsoft, const float* __restrict__ z, uint64_t n,
                     float gamma, float* __restrict__ dz, const TrainDev* st) {
    if (st->halt) return;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x)
        dz[i] = __fmul_rn(dsoft[i], soft_sign_grad_f(z[i], gamma));
}

// C[m][nc] += A[rows][m]^T B[rows][nc] (add_matmul_at, matrix.hpp:121-138):
// each output is one fma chain over the rows in order, from its current
// value; with b1 != null the column sums of B are chained too (b1[j] +=
// B[r][j] in row order, trainer.cpp:231-234). The chains are inherently
// sequential (the reference's rounding order), so the kernel is built for
// latency: one chain per thread, 128 threads = 4 output rows x 32 columns
// (every output gets its own thread), 64-row chunks of A and B double-
// buffered in shared memory with cp.async so the loads of chunk c + 1 run
// under the chains of chunk c.
constexpr int kAtRows = 128;   // rows per stage (== the block size: one A slice per thread)
constexpr int kAtStages = 4;   // cp.async ring depth (3 stages in flight)
constexpr size_t kAtSmem = (size_t)kAtStages * kAtRows * 36 * 4;
struct AtJob {
    const float* A;
    const float* B;
    float* C;
    float* b1;  // optional column sums of B
    uint32_t m, nc;
};
// blockIdx.z selects one of two independent products over the same rows (the
// W2 and W1 gradients of one backward pass run side by side)
__global__ void __launch_bounds__(128) k_add_at(AtJob j0, AtJob j1, uint32_t rows,
                                                const TrainDev* st) {
    if (st->halt) return;
    const AtJob& jb = blockIdx.z ? j1 : j0;
    const float* __restrict__ A = jb.A;
    const float* __restrict__ B = jb.B;
    float* __restrict__ C = jb.C;
    float* __restrict__ b1 = jb.b1;
    const uint32_t m = jb.m, nc = jb.nc;
    if (blockIdx.x * 32 >= nc || blockIdx.y * 4 >= m) return;
    extern __shared__ float at_sm[];  // [stage][kAtRows][4] A, then [stage][kAtRows][32] B
    float* as = at_sm;
    float* bs = at_sm + kAtStages * kAtRows * 4;
    const uint32_t ii = threadIdx.x >> 5, jj = threadIdx.x & 31;
    const uint32_t i = blockIdx.y * 4 + ii, j = blockIdx.x * 32 + jj;
    const bool own = i < m && j < nc;
    const bool bsum = b1 != nullptr && blockIdx.y == 0 && ii == 0 && j < nc;
    float acc = own ? C[(uint64_t)i * nc + j] : 0.0f;
    float bacc = bsum ? b1[j] : 0.0f;
    const uint32_t nch = (rows + kAtRows - 1) / kAtRows;
    // zero-filling 4-byte cp.async (src-size 0 outside the matrices)
    auto cp4 = [](float* dst, const float* src, bool ok) {
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(
                         (uint32_t)__cvta_generic_to_shared(dst)),
                     "l"(src), "r"(ok ? 4 : 0)
                     : "memory");
    };
    const uint32_t bj = blockIdx.x * 32 + (threadIdx.x & 31);
    const uint32_t ai = blockIdx.y * 4 + (threadIdx.x & 3);
    // 16-byte copies when every row slice is 16-byte aligned (m, nc multiples
    // of 4): a quarter of the staging instructions
    const bool v16 = (m & 3u) == 0 && (nc & 3u) == 0;
    auto cp16 = [](float* dst, const float* src, uint32_t bytes) {
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(
                         (uint32_t)__cvta_generic_to_shared(dst)),
                     "l"(src), "r"(bytes)
                     : "memory");
    };
    auto stage = [&](uint32_t c) {  // always commits a group (possibly empty)
        if (c < nch && v16) {
            const uint32_t r0 = c * kAtRows, buf = c % kAtStages;
            float* bsb = bs + (size_t)buf * kAtRows * 32;
            float* asb = as + (size_t)buf * kAtRows * 4;
            const uint32_t q = threadIdx.x & 7, cb = blockIdx.x * 32 + 4 * q;  // 8 x 16 B per B row
#pragma unroll
            for (uint32_t k = 0; k < kAtRows / 16; ++k) {
                const uint32_t r = (threadIdx.x >> 3) + 16 * k;
                const uint32_t left = (r0 + r < rows && cb < nc) ? min(4u, nc - cb) * 4u : 0u;
                cp16(bsb + r * 32 + 4 * q, left ? B + (uint64_t)(r0 + r) * nc + cb : B, left);
            }
            {  // A: one 16-byte slice (4 output rows) per staged row
                const uint32_t r = threadIdx.x;  // kAtRows == blockDim.x
                const uint32_t a0 = blockIdx.y * 4;
                const uint32_t left = (r0 + r < rows && a0 < m) ? min(4u, m - a0) * 4u : 0u;
                cp16(asb + r * 4, left ? A + (uint64_t)(r0 + r) * m + a0 : A, left);
            }
        } else if (c < nch) {
            const uint32_t r0 = c * kAtRows, buf = c % kAtStages;
            float* bsb = bs + (size_t)buf * kAtRows * 32;
            float* asb = as + (size_t)buf * kAtRows * 4;
#pragma unroll 8
            for (uint32_t k = 0; k < kAtRows / 4; ++k) {  // B: rows x 32 columns
                const uint32_t r = (threadIdx.x >> 5) + 4 * k;
                const bool ok = r0 + r < rows && bj < nc;
                cp4(bsb + r * 32 + (threadIdx.x & 31), ok ? B + (uint64_t)(r0 + r) * nc + bj : B, ok);
            }
#pragma unroll
            for (uint32_t k = 0; k < kAtRows / 32; ++k) {  // A: rows x 4 output rows
                const uint32_t r = (threadIdx.x >> 2) + 32 * k;
                const bool ok = r0 + r < rows && ai < m;
                cp4(asb + r * 4 + (threadIdx.x & 3), ok ? A + (uint64_t)(r0 + r) * m + ai : A, ok);
            }
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    for (int c = 0; c < kAtStages - 1; ++c) stage(c);
    for (uint32_t c = 0; c < nch; ++c) {
        asm volatile("cp.async.wait_group %0;" ::"n"(kAtStages - 2) : "memory");
        __syncthreads();
        stage(c + kAtStages - 1);  // refills the slot consumed at c - 1
        const uint32_t buf = c % kAtStages;
        const float* bsb = bs + (size_t)buf * kAtRows * 32 + jj;
        const float* asb = as + (size_t)buf * kAtRows * 4 + ii;
        const uint32_t w = min((uint32_t)kAtRows, rows - c * kAtRows);
        if (w == kAtRows) {
#pragma unroll 16
            for (uint32_t r = 0; r < kAtRows; ++r) {
                const float bv = bsb[r * 32];
                acc = __fmaf_rn(asb[r * 4], bv, acc);
                if (bsum) bacc = __fadd_rn(bacc, bv);
            }
        } else {
            for (uint32_t r = 0; r < w; ++r) {
                const float bv = bsb[r * 32];
                acc = __fmaf_rn(asb[r * 4], bv, acc);
                if (bsum) bacc = __fadd_rn(bacc, bv);
            }
        }
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    if (own) C[(uint64_t)i * nc + j] = acc;
    if (bsum) b1[j] = bacc;
}

// da1 = matmul_bt(dz2, W2) * silu_grad(z1) (trainer.cpp:227-230). W2 staged
// in shared memory with a padded row stride (L + 1: the per-thread rows are
// conflict-free), 32 rows of dz2 per block; thread i keeps the 32 chains of
// its hidden unit (rounded products summed in order, fused tail).
constexpr int kDaRows = 16;
__global__ void __launch_bounds__(128) k_da1(const float* __restrict__ dz2,
                                             const float* __restrict__ w2t,
                                             const float* __restrict__ z1, uint32_t m, uint32_t h,
                                             uint32_t L, float* __restrict__ da1,
                                             const TrainDev* st) {
    if (st->halt) return;
    extern __shared__ float sm[];
    float* ws = sm;                       // [L][h]: W2^T
    float* zs = sm + (size_t)h * L;       // [L][kDaRows] (p-major)
    const uint32_t r0 = blockIdx.x * kDaRows;
    const uint32_t nr = min((uint32_t)kDaRows, m - r0);
    cp_async_f32(ws, w2t, (uint64_t)L * h);  // W2^T [L][h] (kept by k_adamw), contiguous
    for (uint32_t r = 0; r < kDaRows; ++r)  // p-major: zs[p][r] (zero rows past m)
        for (uint32_t p = threadIdx.x; p < L; p += blockDim.x)
            asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(
                             (uint32_t)__cvta_generic_to_shared(zs + p * kDaRows + r)),
                         "l"(r < nr ? dz2 + (uint64_t)(r0 + r) * L + p : dz2), "r"(r < nr ? 4 : 0)
                         : "memory");
    asm volatile("cp.async.commit_group;" ::: "memory");
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    __syncthreads();
    const uint32_t n4 = n4_of(L);
    for (uint32_t i = threadIdx.x; i < h; i += blockDim.x) {
        const float* wr = ws + i;  // W2[i][p] = ws[p * h + i] (consecutive i: no conflicts)
        float acc[kDaRows];
#pragma unroll
        for (int r = 0; r < kDaRows; ++r) acc[r] = 0.0f;
        for (uint32_t p = 0; p < L; ++p) {
            const float wv = wr[(size_t)p * h];
            const float4* zp = reinterpret_cast<const float4*>(zs + p * kDaRows);
            float z[kDaRows];
#pragma unroll
            for (int q = 0; q < kDaRows / 4; ++q) {
                const float4 t = zp[q];
                z[4 * q] = t.x;
                z[4 * q + 1] = t.y;
                z[4 * q + 2] = t.z;
                z[4 * q + 3] = t.w;
            }
            if (p < n4) {
#pragma unroll
                for (int r = 0; r < kDaRows; ++r) acc[r] = __fadd_rn(acc[r], __fmul_rn(z[r], wv));
            } else {
#pragma unroll
                for (int r = 0; r < kDaRows; ++r) acc[r] = __fmaf_rn(z[r], wv, acc[r]);
            }
        }
#pragma unroll
        for (int r = 0; r < kDaRows; ++r)
            if ((uint32_t)r < nr) {
                const uint64_t o = (uint64_t)(r0 + r) * h + i;
                da1[o] = __fmul_rn(acc[r], silu_grad_f(z1[o]));
            }
    }
}

// ------------------------------------------------------------ optimiser
// clip_gradient_norm (trainer.cpp:83-97) + adamw_step's finiteness check and
// bias corrections (:114-121): per-block partial sums of squares (fixed
// order) and non-finite flags, then one small block combines them in order.
// Non-finite after clipping <=> non-finite before (scale <= 1; an infinite
// norm scales finite entries to 0 and infinite ones to NaN), so the flag is
// taken on the raw gradients; k_adamw applies the scale (g * scale, float, as
// the reference's in-place multiply).
constexpr int kNormBlocks = 64;
__global__ void __launch_bounds__(256) k_norm_partial(const float* g, uint64_t n, double* part,
                                                      int* bad, const TrainDev* st) {
    if (st->halt) return;
    __shared__ double s[8];
    __shared__ int s_bad;
    if (threadIdx.x == 0) s_bad = 0;
    __syncthreads();
    double acc = 0.0;
    int b = 0;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const float f = g[i];
        const double v = (double)f;
        acc = __fma_rn(v, v, acc);
        b |= !isfinite(f);
    }
    for (int o = 16; o; o >>= 1) acc = __dadd_rn(acc, __shfl_xor_sync(~0u, acc, o));
    if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = acc;
    if (b) s_bad = 1;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < 8; ++w) t = __dadd_rn(t, s[w]);
        part[blockIdx.x] = t;
        bad[blockIdx.x] = s_bad;
    }
}

__global__ void k_clip(const double* part, const int* bad, double max_norm, const double* bc1_tab,
                       const double* bc2_tab, TrainDev* st) {
    if (st->halt) return;
    __shared__ double s_p[kNormBlocks];
    __shared__ int s_b[kNormBlocks];
    for (int i = threadIdx.x; i < kNormBlocks; i += blockDim.x) {
        s_p[i] = part[i];
        s_b[i] = bad[i];
    }
    __syncthreads();
    if (threadIdx.x) return;
    double t = 0.0;
    int b = 0;
    for (int i = 0; i < kNormBlocks; ++i) {
        t = __dadd_rn(t, s_p[i]);
        b |= s_b[i];
    }
    const double norm = __dsqrt_rn(t);
    st->scale = (max_norm > 0.0 && norm > max_norm) ? __double2float_rn(__ddiv_rn(max_norm, norm)) : 1.0f;
    if (b) {
        st->skip_now = 1;
        st->skipped += 1;
    } else {
        st->skip_now = 0;
        st->step += 1;
        st->bc1 = bc1_tab[st->step];
        st->bc2 = bc2_tab[st->step];
    }
}

// adamw_step's update (trainer.cpp:122-139), f64 moments; decay on
// [0, n_decay0) and [n_decay1, n) (the weight matrices, not b1).
__global__ void k_adamw(float* w, float* g, double* m1, double* m2, uint64_t n,
                        uint64_t n_decay0, uint64_t n_decay1, double lr, double b1, double b2,
                        double eps, double wd, const TrainDev* st, float* w2t, uint32_t h,
                        uint32_t L) {
    if (st->halt) return;
    if (st->skip_now) {  // skipped step: gradients still restart from zero
        for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
             i += (uint64_t)gridDim.x * blockDim.x)
            g[i] = 0.0f;
        return;
    }
    const double bc1 = st->bc1, bc2 = st->bc2;
    const double c1 = __dsub_rn(1.0, b1), c2 = __dsub_rn(1.0, b2);
    const double lwd = __dmul_rn(lr, wd);
    const float sc = st->scale;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const float gr = g[i];
        g[i] = 0.0f;  // the next iteration's gradients start from zero (no memset launch)
        const double gv = (double)(sc != 1.0f ? __fmul_rn(gr, sc) : gr);
        const double m = __fma_rn(b1, m1[i], __dmul_rn(c1, gv));
        const double v = __fma_rn(b2, m2[i], __dmul_rn(__dmul_rn(c2, gv), gv));
        m1[i] = m;
        m2[i] = v;
        const double mhat = __ddiv_rn(m, bc1), vhat = __ddiv_rn(v, bc2);
        const double w_old = (double)w[i];
        double w_new = __dsub_rn(w_old, __ddiv_rn(__dmul_rn(lr, mhat), __dadd_rn(__dsqrt_rn(vhat), eps)));
        if (wd > 0.0 && (i < n_decay0 || i >= n_decay1)) w_new = __fma_rn(-lwd, w_old, w_new);
        const float wf = __double2float_rn(w_new);
        w[i] = wf;
        if (w2t && i >= n_decay1) {  // MLP: keep the transposed W2 copy for k_da1
            const uint64_t e = i - n_decay1;
            w2t[(e % L) * h + e / L] = wf;
        }
    }
}

// ------------------------------------------------------------ host side
uint64_t derive_seed(uint64_t base, uint64_t stream) {  // rng.hpp:10-15
    uint64_t z = base + 0x9E3779B97F4A7C15ULL * (stream + 1);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

// first `take` entries of a random permutation of [0, n), in draw order
// (ranking_loss.cpp:63-75)
std::vector<uint32_t> randperm_take(uint32_t n, uint32_t take, std::mt19937_64& eng) {
    std::vector<uint32_t> perm(n);
    std::iota(perm.begin(), perm.end(), 0u);
    const uint32_t m = std::min(take, n);
    for (uint32_t i = 0; i < m; ++i) {
        std::uniform_int_distribution<uint32_t> pick(i, n - 1);
        std::swap(perm[i], perm[pick(eng)]);
    }
    perm.resize(m);
    return perm;
}

struct Sample {  // one (iteration, batch element) draw
    uint32_t seq = 0;
    std::vector<uint32_t> qrows, top_pos, oth_pos;
    uint32_t k_full = 0;
};

std::string rank_cfg_error(const spl_rank_config& c, uint64_t n) {  // ranking_loss.cpp:13-28
    if (c.beta <= 0.0) return "ranking loss: beta must be positive";
    if (!(c.maskout > 0.0 && c.maskout < 1.0)) return "ranking loss: maskout must lie in (0, 1)";
    const auto k = static_cast<uint32_t>(static_cast<double>(n) * (1.0 - c.maskout));
    if (k == 0) return "ranking loss: top count floored to zero for n=" + std::to_string(n);
    if (c.max_top == 0) return "ranking loss: max_top must be >= 1";
    if (c.max_oth == 0) return "ranking loss: max_oth must be >= 1";
    if (c.query_subsample == 0) return "ranking loss: query_subsample must be >= 1";
    return "";
}

// partition_topk's draws (ranking_loss.cpp:80-116) for a sequence whose
// order covers q_train rows of n keys.
Sample draw_partition(uint32_t q_train, uint32_t n, const spl_rank_config& c, uint64_t seed) {
    Sample s;
    const auto k_full = static_cast<uint32_t>(static_cast<double>(n) * (1.0 - c.maskout));
    const uint32_t oth_full = n - k_full;
    std::mt19937_64 eng(seed);
    s.k_full = k_full;
    s.qrows.resize(q_train);
    std::iota(s.qrows.begin(), s.qrows.end(), 0u);
    if (c.query_subsample > 0 && (uint64_t)c.query_subsample < q_train) {
        s.qrows = randperm_take(q_train, (uint32_t)c.query_subsample, eng);
        std::sort(s.qrows.begin(), s.qrows.end());
    }
    s.top_pos.resize(k_full);
    std::iota(s.top_pos.begin(), s.top_pos.end(), 0u);
    if (c.max_top > 0 && (uint64_t)c.max_top < k_full)
        s.top_pos = randperm_take(k_full, (uint32_t)c.max_top, eng);
    s.oth_pos.resize(oth_full);
    std::iota(s.oth_pos.begin(), s.oth_pos.end(), 0u);
    if (c.max_oth > 0 && (uint64_t)c.max_oth < oth_full)
        s.oth_pos = randperm_take(oth_full, (uint32_t)c.max_oth, eng);
    return s;
}

struct DevBuf {  // owning device allocation list
    std::vector<void*> ptrs;
    ~DevBuf() {
        for (void* p : ptrs) cudaFree(p);
    }
    template <typename T>
    T* get(size_t count) {
        void* p = nullptr;
        if (cudaMalloc(&p, std::max<size_t>(count, 1) * sizeof(T)) != cudaSuccess) return nullptr;
        ptrs.push_back(p);
        return static_cast<T*>(p);
    }
};

}  // namespace

double train_lr_at(uint32_t iter, const spl_train_config& c) {  // trainer.cpp:35-46
    if (c.num_iters == 0) return c.max_lr;
    const uint32_t warmup = std::min(c.warmup_iters, c.num_iters);
    if (iter < warmup) return c.max_lr * static_cast<double>(iter) / static_cast<double>(warmup);
    const uint32_t last = c.num_iters - 1;
    if (last <= warmup) return c.max_lr;
    const double progress = static_cast<double>(iter - warmup) / static_cast<double>(last - warmup);
    // the reference build contracts min + (0.5 (max - min)) (1 + cos) into one fma
    return std::fma(0.5 * (c.max_lr - c.min_lr), 1.0 + std::cos(M_PI * progress), c.min_lr);
}

spl_status train_partition_host(const spl_rank_config& c, uint32_t q_train, uint32_t n,
                                uint64_t seed, uint32_t* rows, uint32_t* top_pos,
                                uint32_t* oth_pos, uint32_t* counts) {
    const Sample s = draw_partition(q_train, n, c, seed);
    std::copy(s.qrows.begin(), s.qrows.end(), rows);
    std::copy(s.top_pos.begin(), s.top_pos.end(), top_pos);
    std::copy(s.oth_pos.begin(), s.oth_pos.end(), oth_pos);
    counts[0] = (uint32_t)s.qrows.size();
    counts[1] = (uint32_t)s.top_pos.size();
    counts[2] = (uint32_t)s.oth_pos.size();
    counts[3] = s.k_full;
    return SPL_OK;
}

// holdout_iou (trainer.cpp:472-518) for the MLP / linear coders: hash codes
// of every key and of the held-out queries (exact encoder K1), Hamming top-k
// (K3, the index shared by all rows: problem stride 0, per-row causal
// n_valid), float top-k of the exact logits, IoU per row, host mean in row
// order.
spl_status holdout_iou_impl(spl_ctx* ctx, int kind, uint32_t d, uint32_t h, uint32_t L,
                            const float* w1, const float* b1, const float* w2, const float* xq,
                            const float* xk, const float* logits, uint32_t q, uint32_t q_train,
                            double rate, double* out, cudaStream_t s) {
    const uint32_t n = q;
    const uint32_t first = q_train < q ? q_train : 0;
    const uint32_t P = q - first;
    uint32_t budget = 0;
    if (spl_status st = spl_budget_from_rate(rate, n, &budget)) return fail(ctx, st, "budget_from_rate");
    DevBuf db;
    uint32_t* nv = db.get<uint32_t>(P);
    uint32_t *ia = db.get<uint32_t>((size_t)P * budget), *ib = db.get<uint32_t>((size_t)P * budget);
    uint32_t *ca = db.get<uint32_t>(P), *cb = db.get<uint32_t>(P);
    double* iou = db.get<double>(P);
    if (!nv || !ia || !ib || !ca || !cb || !iou) return fail(ctx, SPL_E_CUDA, "train: out of device memory");
    std::vector<uint32_t> hv(P);
    for (uint32_t r = 0; r < P; ++r) hv[r] = first + r + 1;  // offsets min(i + 1, n)
    SPL_CUDA_TRY(ctx, cudaMemcpyAsync(nv, hv.data(), P * 4, cudaMemcpyHostToDevice, s));
    if (kind == SPL_HASHER_DOWNPROJ) {
        // kp = K P, qp = Q P (matmul), dp_scores = dot(qp, kp_j), float top-k
        float* dw = db.get<float>((size_t)d * L);
        float* kp = db.get<float>((size_t)n * L);
        float* qp = db.get<float>((size_t)P * L);
        float* sc = db.get<float>((size_t)P * n);
        if (!dw || !kp || !qp || !sc) return fail(ctx, SPL_E_CUDA, "train: out of device memory");
        SPL_CUDA_TRY(ctx, cudaMemcpyAsync(dw, w1, (size_t)d * L * 4, cudaMemcpyHostToDevice, s));
        if (spl_status st = project_launch(ctx, xk, n, d, dw, L, kp, s)) return st;
        if (spl_status st = project_launch(ctx, xq + (size_t)first * d, P, d, dw, L, qp, s)) return st;
        if (spl_status st = causal_logits_launch(ctx, qp, kp, SPL_F32, 0, L, P, nv, 1, n, 1.0f, sc, s))
            return st;
        if (spl_status st = top_k_launch(ctx, sc, 1, P, n, n, budget, ia, s, nv, 1, ca)) return st;
    } else {
        spl_hasher* hs = nullptr;
        if (spl_status st = spl_hasher_create(ctx, kind, 1, d, h, L, w1, b1, w2, &hs)) return st;
        struct HG {
            spl_hasher* h;
            ~HG() { spl_hasher_destroy(h); }
        } guard_{hs};
        const uint32_t W = L / 32;
        uint32_t* kc = db.get<uint32_t>((size_t)n * W);
        uint32_t* qc = db.get<uint32_t>((size_t)P * W);
        if (!kc || !qc) return fail(ctx, SPL_E_CUDA, "train: out of device memory");
        if (spl_status st = spl_encode(ctx, hs, xk, 1, n, SPL_ENCODE_EXACT, kc, s)) return st;
        if (spl_status st = spl_encode(ctx, hs, xq + (size_t)first * d, 1, P, SPL_ENCODE_EXACT, qc, s))
            return st;
        if (spl_status st = hamming_topk_impl(ctx, kc, 0, L, qc, P, nv, 1, n, budget, ia, ca, s)) return st;
    }
    if (spl_status st = top_k_launch(ctx, logits + (size_t)first * n, 1, P, n, n, budget, ib, s, nv, 1, cb))
        return st;
    if (spl_status st = iou_launch(ctx, ia, ca, budget, ib, cb, budget, P, iou, s)) return st;
    std::vector<double> hi(P);
    SPL_CUDA_TRY(ctx, cudaMemcpyAsync(hi.data(), iou, P * 8, cudaMemcpyDeviceToHost, s));
    SPL_CUDA_TRY(ctx, cudaStreamSynchronize(s));
    double sum = 0.0;
    for (double v : hi) sum += v;
    *out = P > 0 ? sum / static_cast<double>(P) : 0.0;
    return SPL_OK;
}

spl_status train_impl(spl_ctx* ctx, int kind, uint32_t d, uint32_t h, uint32_t L, float gamma,
                      float* w1, float* b1, float* w2, uint32_t n_seq, const float* queries,
                      const float* keys, const uint32_t* seq_len, const spl_rank_config& rc,
                      const spl_train_config& tc, bool recon, double* records,
                      double* holdout_iou, uint32_t* skipped, cudaStream_t s) {
    // TrainConfig::validate (trainer.cpp:19-33)
    if (tc.max_lr < 0.0 || tc.min_lr < 0.0 || tc.min_lr > tc.max_lr)
        return fail(ctx, SPL_E_DIMENSION, "TrainConfig: need 0 <= min_lr <= max_lr");
    if (!(tc.adam_beta1 >= 0.0 && tc.adam_beta1 < 1.0 && tc.adam_beta2 >= 0.0 && tc.adam_beta2 < 1.0))
        return fail(ctx, SPL_E_DIMENSION, "TrainConfig: adam betas must lie in [0, 1)");
    if (tc.adam_eps <= 0.0) return fail(ctx, SPL_E_DIMENSION, "TrainConfig: adam_eps must be positive");
    if (tc.weight_decay < 0.0) return fail(ctx, SPL_E_DIMENSION, "TrainConfig: weight_decay must be >= 0");
    if (tc.batch < 1) return fail(ctx, SPL_E_DIMENSION, "TrainConfig: batch must be >= 1");
    if (tc.soft_gamma <= 0.0) return fail(ctx, SPL_E_DIMENSION, "TrainConfig: soft_gamma must be positive");
    if (!(tc.holdout_budget_rate > 0.0 && tc.holdout_budget_rate <= 1.0))
        return fail(ctx, SPL_E_DIMENSION, "TrainConfig: holdout_budget_rate must lie in (0, 1]");
    if (n_seq == 0) return fail(ctx, SPL_E_DIMENSION, "train_hasher: dataset is empty");
    for (uint32_t q = 0; q < n_seq; ++q)
        if (seq_len[q] < 2)
            return fail(ctx, SPL_E_DIMENSION, "train_hasher: sequences need at least two positions");
    const bool mlp = kind == SPL_HASHER_MLP;
    const float sgamma = mlp ? gamma : (float)tc.soft_gamma;  // MlpCoder uses h.gamma
    if (kind == 2 && L == 0) return fail(ctx, SPL_E_DIMENSION, "downproj: width must be >= 1");

    const auto tsetup = std::chrono::steady_clock::now();
    // ---- draws for every iteration (host, the reference's engines)
    const uint32_t iters = tc.num_iters;
    std::vector<uint64_t> off(n_seq + 1, 0);
    for (uint32_t q = 0; q < n_seq; ++q) off[q + 1] = off[q] + seq_len[q];
    auto q_train_of = [&](uint32_t q) {
        const uint32_t rows = seq_len[q];
        const uint32_t holdout = std::min<uint32_t>(tc.holdout_queries, rows / 4);
        uint32_t qt = rows - holdout;
        if (qt < 2) qt = rows;
        return qt;
    };
    std::vector<Sample> draws;
    draws.reserve((size_t)iters * tc.batch);
    std::vector<char> used(n_seq, 0);
    for (uint32_t it = 0; it < iters; ++it) {
        std::mt19937_64 eng(derive_seed(tc.seed, it));
        for (uint32_t b = 0; b < tc.batch; ++b) {
            std::uniform_int_distribution<size_t> pick(0, n_seq - 1);
            const uint32_t sq = (uint32_t)pick(eng);
            const uint64_t part_seed = eng();
            const uint32_t n = seq_len[sq];
            if (!used[sq]) {
                used[sq] = 1;
                const std::string e = rank_cfg_error(rc, n);
                if (!e.empty()) return fail(ctx, SPL_E_DIMENSION, e);
            }
            draws.push_back(draw_partition(q_train_of(sq), n, rc, part_seed));
            draws.back().seq = sq;
        }
    }
    used[0] = 1;  // the holdout IoU reads sequence 0

    // ---- device state
    DevBuf db;
    const uint64_t n1 = (uint64_t)d * (mlp ? h : L), nb = mlp ? h : 0, n2 = mlp ? (uint64_t)h * L : 0;
    const uint64_t np = n1 + nb + n2;
    float* dP = db.get<float>(np);
    float* dG = db.get<float>(np);
    double* dM = db.get<double>(np);
    double* dV = db.get<double>(np);
    TrainDev* dst = db.get<TrainDev>(1);
    double* drec = db.get<double>((size_t)iters * 3 + 3);
    if (!dP || !dG || !dM || !dV || !dst || !drec) return fail(ctx, SPL_E_CUDA, "train: out of device memory");
    SPL_CUDA_TRY(ctx, cudaMemcpyAsync(dP, w1, n1 * 4, cudaMemcpyHostToDevice, s));
    if (mlp) {
        SPL_CUDA_TRY(ctx, cudaMemcpyAsync(dP + n1, b1, nb * 4, cudaMemcpyHostToDevice, s));
        SPL_CUDA_TRY(ctx, cudaMemcpyAsync(dP + n1 + nb, w2, n2 * 4, cudaMemcpyHostToDevice, s));
    }
    SPL_CUDA_TRY(ctx, cudaMemsetAsync(dM, 0, np * 8, s));
    SPL_CUDA_TRY(ctx, cudaMemsetAsync(dG, 0, np * 4, s));  // k_adamw re-zeroes it every step
    SPL_CUDA_TRY(ctx, cudaMemsetAsync(dV, 0, np * 8, s));
    SPL_CUDA_TRY(ctx, cudaMemsetAsync(dst, 0, sizeof(TrainDev), s));
    SPL_CUDA_TRY(ctx, cudaMemsetAsync(drec, 0, ((size_t)iters * 3 + 3) * 8, s));
    // bias corrections 1 - beta^t for every step t the run can reach (host
    // std::pow, as adamw_step computes them)
    std::vector<double> bc1(iters + 2), bc2(iters + 2);
    for (uint32_t t = 0; t < iters + 2; ++t) {
        bc1[t] = 1.0 - std::pow(tc.adam_beta1, static_cast<double>(t));
        bc2[t] = 1.0 - std::pow(tc.adam_beta2, static_cast<double>(t));
    }
    double* dbc1 = db.get<double>(iters + 2);
    double* dbc2 = db.get<double>(iters + 2);
    double* npart = db.get<double>(kNormBlocks);
    int* nbad = db.get<int>(kNormBlocks);
    if (!dbc1 || !dbc2 || !npart || !nbad) return fail(ctx, SPL_E_CUDA, "train: out of device memory");
    SPL_CUDA_TRY(ctx, cudaMemcpyAsync(dbc1, bc1.data(), bc1.size() * 8, cudaMemcpyHostToDevice, s));
    SPL_CUDA_TRY(ctx, cudaMemcpyAsync(dbc2, bc2.data(), bc2.size() * 8, cudaMemcpyHostToDevice, s));

    // ---- per-sequence preparation: inputs, exact logits, order (prepare_sequence)
    struct Prep {
        float* x_q = nullptr;
        float* x_k = nullptr;
        float* logits = nullptr;
        uint32_t* order = nullptr;
        uint32_t q_train = 0;
    };
    std::vector<Prep> prep(n_seq);
    const float scale = 1.0f / std::sqrt(static_cast<float>(d));
    uint32_t max_n = 0;
    for (uint32_t q = 0; q < n_seq; ++q) {
        if (!used[q]) continue;
        const uint32_t n = seq_len[q];
        max_n = std::max(max_n, n);
        Prep& p = prep[q];
        p.q_train = q_train_of(q);
        p.x_q = db.get<float>((size_t)n * d);
        p.x_k = db.get<float>((size_t)n * d);
        p.logits = db.get<float>((size_t)n * n);
        p.order = db.get<uint32_t>((size_t)p.q_train * n);
        if (!p.x_q || !p.x_k || !p.logits || !p.order) return fail(ctx, SPL_E_CUDA, "train: out of device memory");
        SPL_CUDA_TRY(ctx, cudaMemcpyAsync(p.x_q, queries + off[q] * d, (size_t)n * d * 4, cudaMemcpyHostToDevice, s));
        SPL_CUDA_TRY(ctx, cudaMemcpyAsync(p.x_k, keys + off[q] * d, (size_t)n * d * 4, cudaMemcpyHostToDevice, s));
        k_logits<<<dim3((n + 63) / 64, (n + 63) / 64), 256, 0, s>>>(p.x_q, p.x_k, n, n, d, scale, p.logits);
        if (spl_status st = after_launch(ctx, "k_logits")) return st;
        // build_topk_order: bitonic chunks of C keys in shared memory, then
        // merge passes in global memory for rows longer than one chunk
        uint32_t C = 1;
        while (C < n && C < kMaxSortKeys) C <<= 1;
        const uint32_t nch = (n + C - 1) / C;
        const size_t smem = (size_t)C * 8;
        SPL_CUDA_TRY(ctx, cudaFuncSetAttribute(k_order, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        if (nch == 1) {
            k_order<<<dim3(1, p.q_train), 1024, smem, s>>>(p.logits, n, C, 0, p.order, nullptr);
            if (spl_status st = after_launch(ctx, "k_order")) return st;
        } else {
            const uint64_t rowlen = (uint64_t)nch * C;
            const uint32_t rb = (uint32_t)std::max<uint64_t>(1, std::min<uint64_t>(p.q_train, (1ull << 31) / (16 * rowlen)));
            unsigned long long* ra = db.get<unsigned long long>((size_t)rb * rowlen);
            unsigned long long* rbuf = db.get<unsigned long long>((size_t)rb * rowlen);
            if (!ra || !rbuf) return fail(ctx, SPL_E_CUDA, "train: out of device memory");
            for (uint32_t r0 = 0; r0 < p.q_train; r0 += rb) {
                const uint32_t rows = std::min(rb, p.q_train - r0);
                k_order<<<dim3(nch, rows), 1024, smem, s>>>(p.logits, n, C, r0, nullptr, ra);
                if (spl_status st = after_launch(ctx, "k_order")) return st;
                unsigned long long *src = ra, *dstb = rbuf;
                for (uint64_t R = C; R < rowlen; R <<= 1) {
                    const uint64_t total = (uint64_t)rows * rowlen;
                    k_order_merge<<<(unsigned)std::min<uint64_t>((total + 255) / 256, 148 * 16), 256, 0, s>>>(
                        src, dstb, rowlen, R, total);
                    if (spl_status st = after_launch(ctx, "k_order_merge")) return st;
                    std::swap(src, dstb);
                }
                const uint64_t tot = (uint64_t)rows * n;
                k_order_extract<<<(unsigned)std::min<uint64_t>((tot + 255) / 256, 148 * 16), 256, 0, s>>>(
                    src, rowlen, n, r0, rows, p.order);
                if (spl_status st = after_launch(ctx, "k_order_extract")) return st;
            }
        }
    }

    // ---- per-step buffers (sized for the largest draw)
    uint32_t maxQ = 1, maxT = 1, maxO = 1;
    for (const Sample& w : draws) {
        maxQ = std::max<uint32_t>(maxQ, (uint32_t)w.qrows.size());
        maxT = std::max<uint32_t>(maxT, (uint32_t)w.top_pos.size());
        maxO = std::max<uint32_t>(maxO, (uint32_t)w.oth_pos.size());
    }
    auto dk_smem = [&](uint32_t qs) { return ((size_t)qs * L + (size_t)kDkKeys * qs) * 4; };
    const bool dk_staged = dk_smem(maxQ) <= 200 * 1024;
    if (dk_staged)
        SPL_CUDA_TRY(ctx, cudaFuncSetAttribute(k_dsoft_keys, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dk_smem(maxQ)));
    const size_t grad_smem = (size_t)(maxT + maxO) * 16;
    // Limits of the GPU trainer (the reference streams each query and has
    // none): the top + other keys of one draw are staged in one block's shared
    // memory, and the pair gradients are materialised as maxQ x maxT x maxO
    // doubles. Both are stated here rather than failing inside an allocation.
    if (grad_smem > 200 * 1024)
        return fail(ctx, SPL_E_DIMENSION,
                    "train_hasher: GPU trainer limit: max_top + max_oth = " +
                        std::to_string(maxT + maxO) +
                        " sampled keys per query exceed one block's shared memory (<= 12800); "
                        "set RankingLossConfig max_top / max_oth");
    {
        size_t free_b = 0, total_b = 0;
        const size_t gpair_b = (size_t)maxQ * maxT * maxO * sizeof(double);
        if (cudaMemGetInfo(&free_b, &total_b) == cudaSuccess && gpair_b > free_b / 2)
            return fail(ctx, SPL_E_DIMENSION,
                        "train_hasher: GPU trainer limit: the pair-gradient buffer (queries x top x "
                        "other = " + std::to_string(gpair_b >> 20) +
                            " MiB of doubles) exceeds half the free device memory; set "
                            "query_subsample / max_top / max_oth");
    }
    SPL_CUDA_TRY(ctx, cudaFuncSetAttribute(k_rank_grad, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)grad_smem));
    const uint64_t pair_blocks = std::max<uint64_t>(
        ((uint64_t)maxT * maxO + kPairThreads * kPairsPerThread - 1) / (kPairThreads * kPairsPerThread),
        (max_n + 255) / 256);  // also the reconstruction loss's blocks per query
    const uint32_t hw = mlp ? h : 1;
    float *z1q = db.get<float>((size_t)maxQ * hw), *a1q = db.get<float>((size_t)maxQ * hw);
    float *z2q = db.get<float>((size_t)maxQ * L), *sfq = db.get<float>((size_t)maxQ * L);
    float *z1k = db.get<float>((size_t)max_n * hw), *a1k = db.get<float>((size_t)max_n * hw);
    float *z2k = db.get<float>((size_t)max_n * L), *sfk = db.get<float>((size_t)max_n * L);
    float *dsq = db.get<float>((size_t)maxQ * L), *dsk = db.get<float>((size_t)max_n * L);
    float *dz = db.get<float>((size_t)std::max(maxQ, max_n) * L);
    float *da1 = db.get<float>((size_t)std::max(maxQ, max_n) * hw);
    float *Gm = db.get<float>((size_t)max_n * maxQ);
    double* bcv = db.get<double>((size_t)maxQ * (maxT + maxO));
    double* gpair = db.get<double>((size_t)maxQ * maxT * maxO);
    double* lpart = db.get<double>((size_t)maxQ * pair_blocks);
    unsigned long long* vpart = db.get<unsigned long long>((size_t)maxQ * pair_blocks);
    uint32_t *top_idx = db.get<uint32_t>((size_t)maxQ * maxT), *oth_idx = db.get<uint32_t>((size_t)maxQ * maxO);
    // every draw's index lists, uploaded once
    std::vector<uint64_t> doff(draws.size() + 1, 0);
    for (size_t i = 0; i < draws.size(); ++i)
        doff[i + 1] = doff[i] + draws[i].qrows.size() + draws[i].top_pos.size() + draws[i].oth_pos.size();
    std::vector<uint32_t> hdraw(doff.back());
    for (size_t i = 0; i < draws.size(); ++i) {
        uint32_t* p = hdraw.data() + doff[i];
        p = std::copy(draws[i].qrows.begin(), draws[i].qrows.end(), p);
        p = std::copy(draws[i].top_pos.begin(), draws[i].top_pos.end(), p);
        std::copy(draws[i].oth_pos.begin(), draws[i].oth_pos.end(), p);
    }
    uint32_t* ddraw = db.get<uint32_t>(hdraw.size());
    if (!z1q || !a1q || !z2q || !sfq || !z1k || !a1k || !z2k || !sfk || !dsq || !dsk || !dz || !da1 ||
        !Gm || !bcv || !gpair || !lpart || !vpart || !top_idx || !oth_idx || !ddraw)
        return fail(ctx, SPL_E_CUDA, "train: out of device memory");
    if (!hdraw.empty())
        SPL_CUDA_TRY(ctx, cudaMemcpyAsync(ddraw, hdraw.data(), hdraw.size() * 4, cudaMemcpyHostToDevice, s));

    float* gW1 = dG;
    float* gB1 = dG + n1;
    float* gW2 = dG + n1 + nb;
    const float* W1 = dP;
    const float* B1 = dP + n1;
    const float* W2 = dP + n1 + nb;
    float* W2T = nullptr;  // MLP: W2 transposed [L][h] for k_da1 (k_adamw keeps it current)
    if (mlp) {
        W2T = db.get<float>((size_t)h * L);
        if (!W2T) return fail(ctx, SPL_E_CUDA, "train: out of device memory");
        k_transpose<<<(unsigned)std::min<uint64_t>(((uint64_t)h * L + 255) / 256, 1024), 256, 0, s>>>(
            W2, h, L, W2T);
        if (spl_status st = after_launch(ctx, "k_transpose")) return st;
    }
    // forward: weights staged in shared memory when they fit (one block/SM)
    const size_t wbytes = (mlp ? std::max((size_t)d * h, (size_t)h * L) : (size_t)d * L) * 4;
    const size_t fwd_base = (size_t)kFwdRows * (d + (mlp ? h : 0)) * 4;
    const bool wsmem = fwd_base + wbytes <= 220 * 1024;
    const size_t fwd_smem = fwd_base + (wsmem ? wbytes : 0);
    auto fwd_attr = [&](const void* fn) -> spl_status {
        SPL_CUDA_TRY(ctx, cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fwd_smem));
        return SPL_OK;
    };
    {
        const void* fns[6] = {(const void*)k_forward<SPL_HASHER_MLP, true>, (const void*)k_forward<SPL_HASHER_MLP, false>,
                              (const void*)k_forward<SPL_HASHER_LINEAR, true>, (const void*)k_forward<SPL_HASHER_LINEAR, false>,
                              (const void*)k_forward<2, true>, (const void*)k_forward<2, false>};
        for (const void* f : fns)
            if (spl_status st = fwd_attr(f)) return st;
    }
    auto fwd = [&](const float* x, const uint32_t* rows, uint32_t m, float* a, float* b, float* c,
                   float* sf, float* xcopy) -> spl_status {
        const dim3 grid((m + kFwdRows - 1) / kFwdRows);
#define SPL_FWD(K_, WS_) k_forward<K_, WS_><<<grid, kFwdThreads, fwd_smem, s>>>(x, rows, m, d, K_ == SPL_HASHER_MLP ? h : 0, L, W1, K_ == SPL_HASHER_MLP ? B1 : nullptr, K_ == SPL_HASHER_MLP ? W2 : nullptr, sgamma, a, b, c, sf, dst, xcopy)
        if (kind == SPL_HASHER_MLP) { if (wsmem) SPL_FWD(SPL_HASHER_MLP, true); else SPL_FWD(SPL_HASHER_MLP, false); }
        else if (kind == SPL_HASHER_LINEAR) { if (wsmem) SPL_FWD(SPL_HASHER_LINEAR, true); else SPL_FWD(SPL_HASHER_LINEAR, false); }
        else { if (wsmem) SPL_FWD(2, true); else SPL_FWD(2, false); }
#undef SPL_FWD
        return after_launch(ctx, "k_forward");
    };
    // backward of one side (trainer.cpp:219-236 / :252-258 / :279-282);
    // x rows are gathered (queries) or identity (keys)
    float* xg = db.get<float>((size_t)maxQ * d);  // gathered query inputs for add_at
    if (!xg) return fail(ctx, SPL_E_CUDA, "train: out of device memory");
    SPL_CUDA_TRY(ctx, cudaFuncSetAttribute(k_add_at, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kAtSmem));
    const size_t da1_smem = mlp ? ((size_t)h * L + (size_t)kDaRows * L) * 4 : 0;
    if (da1_smem > 220 * 1024)
        return fail(ctx, SPL_E_DIMENSION, "train_hasher: hidden x code width too large for the GPU trainer");
    if (mlp)
        SPL_CUDA_TRY(ctx, cudaFuncSetAttribute(k_da1, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)da1_smem));
    auto bwd = [&](const float* x, uint32_t m, const float* z1, const float* a1, const float* z2,
                   const float* dsoft) -> spl_status {
        const uint64_t ne = (uint64_t)m * L;
        const unsigned eg = (unsigned)std::min<uint64_t>((ne + 255) / 256, 4096);
        const float* dzp = dsoft;
        if (kind != 2) {
            k_dz<<<eg, 256, 0, s>>>(dsoft, z2, ne, sgamma, dz, dst);
            if (spl_status st = after_launch(ctx, "k_dz")) return st;
            dzp = dz;
        }
        if (mlp) {
            // da1 first, then W2 += a1^T dz2 and W1 += x^T da1 (+ b1) in one
            // launch: independent accumulators, so the order between them is free
            k_da1<<<(m + kDaRows - 1) / kDaRows, 128, da1_smem, s>>>(dzp, W2T, z1, m, h, L, da1, dst);
            if (spl_status st = after_launch(ctx, "k_da1")) return st;
            const AtJob jw2{a1, dzp, gW2, nullptr, h, L}, jw1{x, da1, gW1, gB1, d, h};
            const dim3 grid((std::max(L, h) + 31) / 32, (std::max(h, d) + 3) / 4, 2);
            k_add_at<<<grid, 128, kAtSmem, s>>>(jw2, jw1, m, dst);
            return after_launch(ctx, "k_add_at");
        }
        const AtJob jp{x, dzp, gW1, nullptr, d, L};
        k_add_at<<<dim3((L + 31) / 32, (d + 3) / 4, 1), 128, kAtSmem, s>>>(jp, jp, m, dst);
        return after_launch(ctx, "k_add_at");
    };
    const float invb = tc.batch > 1 ? (float)(1.0 / tc.batch) : 1.0f;
    // device time of the loop (spl_train_last_loop_ms); SPL_TRAIN_PROFILE=1
    // also prints host enqueue vs device time and the setup / holdout costs
    const char* prof = getenv("SPL_TRAIN_PROFILE");
    cudaEvent_t pe[2];
    SPL_CUDA_TRY(ctx, cudaEventCreate(&pe[0]));
    SPL_CUDA_TRY(ctx, cudaEventCreate(&pe[1]));
    struct EvGuard {
        cudaEvent_t* e;
        ~EvGuard() {
            cudaEventDestroy(e[0]);
            cudaEventDestroy(e[1]);
        }
    } evg_{pe};
    SPL_CUDA_TRY(ctx, cudaEventRecord(pe[0], s));
    const std::chrono::steady_clock::time_point pt0 = std::chrono::steady_clock::now();
    for (uint32_t it = 0; it < iters; ++it) {
        const double lr = train_lr_at(it, tc);
        for (uint32_t b = 0; b < tc.batch; ++b) {
            const size_t di = (size_t)it * tc.batch + b;
            const Sample& w = draws[di];
            const Prep& p = prep[w.seq];
            const uint32_t n = seq_len[w.seq];
            const uint32_t Qs = (uint32_t)w.qrows.size(), T = (uint32_t)w.top_pos.size(),
                           O = (uint32_t)w.oth_pos.size();
            const uint32_t* qrows = ddraw + doff[di];
            const uint32_t* tpos = qrows + Qs;
            const uint32_t* opos = tpos + T;
            SPL_CUDA_TRY(ctx, cudaMemsetAsync(Gm, 0, (size_t)n * Qs * 4, s));
            k_partition<<<Qs, 256, 0, s>>>(p.order, n, w.k_full, qrows, tpos, T, opos, O, top_idx, oth_idx, dst);
            if (spl_status st = after_launch(ctx, "k_partition")) return st;
            if (spl_status st = fwd(p.x_q, qrows, Qs, z1q, a1q, z2q, sfq, xg)) return st;
            if (spl_status st = fwd(p.x_k, nullptr, n, z1k, a1k, z2k, sfk, nullptr)) return st;
            if (!recon) {
                k_rank_dots<<<dim3(Qs, (T + O + 127) / 128), 128, (size_t)L * 4, s>>>(
                    sfq, sfk, L, top_idx, T, oth_idx, O, bcv, dst, it);
                if (spl_status st = after_launch(ctx, "k_rank_dots")) return st;
                const uint32_t pb = (uint32_t)(((uint64_t)T * O + kPairThreads * kPairsPerThread - 1) /
                                               (kPairThreads * kPairsPerThread));
                k_rank_pairs<<<dim3(Qs, pb), kPairThreads, 0, s>>>(bcv, top_idx, T, oth_idx, O, rc.beta,
                                                                    rc.alpha, gpair, lpart, vpart, dst);
                if (spl_status st = after_launch(ctx, "k_rank_pairs")) return st;
                k_rank_grad<<<Qs, 256, (size_t)(T + O) * 16, s>>>(
                    sfk, L, top_idx, T, oth_idx, O, Qs, gpair, Gm, dsq, dst);
                if (spl_status st = after_launch(ctx, "k_rank_grad")) return st;
                k_loss_finalize<<<1, 256, 0, s>>>(lpart, vpart, Qs * pb, b, tc.batch, it, drec, dst, 0.0);
                if (spl_status st = after_launch(ctx, "k_loss_finalize")) return st;
            } else {
                // count = sum over the selected rows of their causal offsets
                double count = 0.0;
                for (uint32_t r : w.qrows) count += (double)std::min(r + 1, n);
                const uint32_t yb = std::min<uint32_t>((n + 255) / 256, (uint32_t)pair_blocks);
                k_recon<<<dim3(Qs, yb), 256, (size_t)L * 4, s>>>(sfq, sfk, L, p.logits, n, qrows, Qs,
                                                                 2.0 / count, Gm, lpart, dst);
                if (spl_status st = after_launch(ctx, "k_recon")) return st;
                k_recon_dq<<<Qs, 128, 0, s>>>(Gm, sfk, L, n, qrows, Qs, invb, dsq, dst);
                if (spl_status st = after_launch(ctx, "k_recon_dq")) return st;
                SPL_CUDA_TRY(ctx, cudaMemsetAsync(vpart, 0, (size_t)Qs * yb * 8, s));
                k_loss_finalize<<<1, 256, 0, s>>>(lpart, vpart, Qs * yb, b, tc.batch, it, drec, dst, count);
                if (spl_status st = after_launch(ctx, "k_loss_finalize")) return st;
            }
            if (dk_staged)
                k_dsoft_keys<<<(n + kDkKeys - 1) / kDkKeys, 256, dk_smem(Qs), s>>>(Gm, sfq, Qs, n, L, invb, dsk, dst);
            else
                k_dsoft_keys_flat<<<(unsigned)(((uint64_t)n * L + 255) / 256), 256, 0, s>>>(Gm, sfq, Qs, n, L, invb, dsk, dst);
            if (spl_status st = after_launch(ctx, "k_dsoft_keys")) return st;
            if (invb != 1.0f && !recon) {
                k_scale<<<(Qs * L + 255) / 256, 256, 0, s>>>(dsq, (uint64_t)Qs * L, invb, dst);
                if (spl_status st = after_launch(ctx, "k_scale")) return st;
            }
            if (spl_status st = bwd(xg, Qs, z1q, a1q, z2q, dsq)) return st;
            if (spl_status st = bwd(p.x_k, n, z1k, a1k, z2k, dsk)) return st;
        }
        k_norm_partial<<<kNormBlocks, 256, 0, s>>>(dG, np, npart, nbad, dst);
        if (spl_status st = after_launch(ctx, "k_norm_partial")) return st;
        k_clip<<<1, kNormBlocks, 0, s>>>(npart, nbad, tc.grad_clip, dbc1, dbc2, dst);
        if (spl_status st = after_launch(ctx, "k_clip")) return st;
        k_adamw<<<(unsigned)std::min<uint64_t>((np + 255) / 256, 1184), 256, 0, s>>>(
            dP, dG, dM, dV, np, n1, n1 + nb, lr, tc.adam_beta1, tc.adam_beta2, tc.adam_eps,
            tc.weight_decay, dst, mlp ? W2T : nullptr, h, L);
        if (spl_status st = after_launch(ctx, "k_adamw")) return st;
    }

    {
        const double host_ms =
            std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - pt0).count();
        SPL_CUDA_TRY(ctx, cudaEventRecord(pe[1], s));
        SPL_CUDA_TRY(ctx, cudaEventSynchronize(pe[1]));
        float dev_ms = 0;
        SPL_CUDA_TRY(ctx, cudaEventElapsedTime(&dev_ms, pe[0], pe[1]));
        ctx->last_train_loop_ms = dev_ms;
        if (prof && *prof == '1')
            fprintf(stderr, "train loop: %u iters, host enqueue %.3f ms, device %.3f ms (%.3f ms/iter)\n",
                    iters, host_ms, dev_ms, iters ? dev_ms / iters : 0.0);
    }
    // ---- results: weights (also on the error paths, as the reference's
    // in-place hasher), records, then the holdout IoU
    TrainDev hs{};
    SPL_CUDA_TRY(ctx, cudaMemcpyAsync(&hs, dst, sizeof(TrainDev), cudaMemcpyDeviceToHost, s));
    SPL_CUDA_TRY(ctx, cudaMemcpyAsync(w1, dP, n1 * 4, cudaMemcpyDeviceToHost, s));
    if (mlp) {
        SPL_CUDA_TRY(ctx, cudaMemcpyAsync(b1, dP + n1, nb * 4, cudaMemcpyDeviceToHost, s));
        SPL_CUDA_TRY(ctx, cudaMemcpyAsync(w2, dP + n1 + nb, n2 * 4, cudaMemcpyDeviceToHost, s));
    }
    if (records && iters)
        SPL_CUDA_TRY(ctx, cudaMemcpyAsync(records, drec, (size_t)iters * 3 * 8, cudaMemcpyDeviceToHost, s));
    SPL_CUDA_TRY(ctx, cudaStreamSynchronize(s));
    if (hs.halt == HALT_EMPTY)
        return fail(ctx, SPL_E_EMPTY_PAIRS, "ranking loss: no causally valid pairs to rank");
    if (hs.halt == HALT_NONFINITE)
        return fail(ctx, SPL_E_NUMERIC, "train_hasher: loss became non-finite at iteration " +
                                            std::to_string(hs.halt_iter));
    if (records)
        for (uint32_t it = 0; it < iters; ++it) records[3 * (size_t)it + 2] = train_lr_at(it, tc);
    if (skipped) *skipped = hs.skipped;
    const auto th0 = std::chrono::steady_clock::now();
    if (holdout_iou) {
        spl_status st = holdout_iou_impl(ctx, kind, d, h, L, w1, b1, w2, prep[0].x_q, prep[0].x_k,
                                         prep[0].logits, seq_len[0], prep[0].q_train,
                                         tc.holdout_budget_rate, holdout_iou, s);
        if (st) return st;
    }
    if (prof && *prof == '1')
        fprintf(stderr, "train: setup %.3f ms, holdout %.3f ms\n",
                std::chrono::duration<double, std::milli>(pt0 - tsetup).count(),
                std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - th0).count());
    return SPL_OK;
}

}  // namespace spl

// ------------------------------------------------------------ C-ABI
extern "C" spl_status spl_train_hasher(spl_ctx* ctx, int kind, uint32_t d, uint32_t h, uint32_t L,
                                       float gamma, float* w1, float* b1, float* w2,
                                       uint32_t n_seq, const float* queries, const float* keys,
                                       const uint32_t* seq_len, const spl_rank_config* rank,
                                       const spl_train_config* train, int loss_kind,
                                       double* records, double* holdout_iou, uint32_t* skipped,
                                       void* stream) {
    if (!ctx) return SPL_E_STATE;
    if (!rank || !train || !w1 || (kind == SPL_HASHER_MLP && (!b1 || !w2)) ||
        (n_seq && (!queries || !keys || !seq_len)))
        return spl::fail(ctx, SPL_E_STATE, "train_hasher: null pointer");
    if (kind != SPL_HASHER_MLP && kind != SPL_HASHER_LINEAR && kind != SPL_HASHER_DOWNPROJ)
        return spl::fail(ctx, SPL_E_DIMENSION, "train_hasher: unknown hasher kind");
    if (d == 0 || L == 0 || (kind == SPL_HASHER_MLP && h == 0))
        return spl::fail(ctx, SPL_E_DIMENSION, "train_hasher: dimensions must be >= 1");
    if (kind != SPL_HASHER_DOWNPROJ && L % 32 != 0)
        return spl::fail(ctx, SPL_E_DIMENSION, "train_hasher: code bits must be a multiple of 32");
    if (loss_kind != SPL_TRAIN_LOSS_RANKING && loss_kind != SPL_TRAIN_LOSS_RECONSTRUCTION)
        return spl::fail(ctx, SPL_E_DIMENSION, "train_hasher: unknown loss kind");
    return spl::train_impl(ctx, kind, d, h, L, gamma, w1, b1, w2, n_seq, queries, keys, seq_len,
                           *rank, *train, loss_kind == SPL_TRAIN_LOSS_RECONSTRUCTION, records,
                           holdout_iou, skipped, static_cast<cudaStream_t>(stream));
}

extern "C" spl_status spl_train_partition_host(const spl_rank_config* rank, uint32_t q_train,
                                               uint32_t n, uint64_t seed, uint32_t* rows,
                                               uint32_t* top_pos, uint32_t* oth_pos,
                                               uint32_t* counts) {
    if (!rank || !rows || !top_pos || !oth_pos || !counts) return SPL_E_STATE;
    return spl::train_partition_host(*rank, q_train, n, seed, rows, top_pos, oth_pos, counts);
}

extern "C" double spl_train_last_loop_ms(const spl_ctx* ctx) {
    return ctx ? ctx->last_train_loop_ms : 0.0;
}

extern "C" double spl_train_lr_at(uint32_t iter, const spl_train_config* train) {
    return train ? spl::train_lr_at(iter, *train) : 0.0;
}
