// K4/K5 — sparse decode attention over the retrieved rows (sm_100a).
//
// Replaces sparse_attention (attention_eval.cpp:234-264) + attend_subset
// (:54-78): per problem, softmax(q K_S^T * scale) V_S over S = picked U {own}
// (the own row n_valid - 1 is always attended, :249-260). Flash-decoding:
// the row list is split across CTAs (grid = splits x problems); each warp
// gathers 8 rows at a time (lane owns d/32 contiguous dims, one coalesced
// 8 B (bf16) / 16 B (f32) load per lane per row), keeps an online-softmax
// (m, l, o) in fp32 registers (log2 domain: q is pre-scaled by
// scale*log2(e)), warps merge in shared memory, and the CTA that finishes a
// problem's last split performs the log-sum-exp combine (K5) — one launch.
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <string>

#include "spl_launch.cuh"

namespace spl {

constexpr int kAttThreads = 128;
constexpr int kAttWarps = kAttThreads / 32;
constexpr int kGroup = 8;  // rows in flight per warp

// Raw (undecoded) row slice of one lane: E elements of a K or V row. Loaded
// as one coalesced vector per lane (warp = one full row), decoded to fp32 at
// use, so the double buffer costs E/2 (bf16) or E (f32) registers per row.
template <int E, typename KV>
struct Raw;
template <int E>
struct Raw<E, __nv_bfloat16> {
    static_assert(E == 1 || E == 2 || E == 4 || E == 8, "E");
    uint32_t u[(E + 1) / 2];
    __device__ __forceinline__ void load(const __nv_bfloat16* row, int lane) {
        const __nv_bfloat16* p = row + lane * E;
        if constexpr (E == 8) {
            const uint4 v = __ldg(reinterpret_cast<const uint4*>(p));
            u[0] = v.x; u[1] = v.y; u[2] = v.z; u[3] = v.w;
        } else if constexpr (E == 4) {
            const uint2 v = __ldg(reinterpret_cast<const uint2*>(p));
            u[0] = v.x; u[1] = v.y;
        } else if constexpr (E == 2) {
            u[0] = __ldg(reinterpret_cast<const unsigned int*>(p));
        } else {
            u[0] = __ldg(reinterpret_cast<const unsigned short*>(p));
        }
    }
    __device__ __forceinline__ float get(int e) const {
        const uint32_t w = u[e / 2];
        return __uint_as_float((e & 1) ? (w & 0xffff0000u) : (w << 16));
    }
};
template <int E>
struct Raw<E, float> {
    float f[E];
    __device__ __forceinline__ void load(const float* row, int lane) {
        const float* p = row + lane * E;
        if constexpr (E % 4 == 0) {
#pragma unroll
            for (int i = 0; i < E; i += 4) {
                const float4 v = __ldg(reinterpret_cast<const float4*>(p + i));
                f[i] = v.x; f[i + 1] = v.y; f[i + 2] = v.z; f[i + 3] = v.w;
            }
        } else if constexpr (E == 2) {
            const float2 v = __ldg(reinterpret_cast<const float2*>(p));
            f[0] = v.x; f[1] = v.y;
        } else {
            f[0] = __ldg(p);
        }
    }
    __device__ __forceinline__ float get(int e) const { return f[e]; }
};

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

constexpr uint32_t kInv = 0xFFFFFFFFu;
constexpr uint32_t kWarpRows = 64;  // rows per warp per split (2 indices per lane)

// rows per in-flight group: 8, or 4 when a lane's slice of a row is >= 32 B
template <int E, typename KV>
constexpr int group_rows() {
    return E * (int)sizeof(KV) >= 32 ? 4 : kGroup;
}

template <int E, typename KV>
struct Group {
    static constexpr int G = group_rows<E, KV>();
    Raw<E, KV> k[G], v[G];
    uint32_t row[G];
    __device__ __forceinline__ void issue(uint32_t rid, int sub, const KV* kb, const KV* vb,
                                          int lane) {
#pragma unroll
        for (int r = 0; r < G; ++r) {
            row[r] = __shfl_sync(0xffffffffu, rid, sub * G + r);
            if (row[r] != kInv) {
                k[r].load(kb + (uint64_t)row[r] * (32 * E), lane);
                v[r].load(vb + (uint64_t)row[r] * (32 * E), lane);
            }
        }
    }
};

template <int E, typename KV>
__device__ __forceinline__ void consume(const Group<E, KV>& g, const float* qv, float& m, float& l,
                                        float* o) {
    constexpr int G = Group<E, KV>::G;
    float s[G];
    float gmax = -INFINITY;
#pragma unroll
    for (int r = 0; r < G; ++r) {
        float part = 0.0f;
#pragma unroll
        for (int e = 0; e < E; ++e) part = fmaf(qv[e], g.k[r].get(e), part);
        part = warp_sum(part);
        s[r] = g.row[r] != kInv ? part : -INFINITY;
        gmax = fmaxf(gmax, s[r]);
    }
    if (gmax == -INFINITY) return;
    const float m_new = fmaxf(m, gmax);
    const float corr = exp2f(m - m_new);  // m = -inf -> 0
    l *= corr;
#pragma unroll
    for (int e = 0; e < E; ++e) o[e] *= corr;
#pragma unroll
    for (int r = 0; r < G; ++r) {
        if (g.row[r] == kInv) continue;  // never touch unloaded registers
        const float w = exp2f(s[r] - m_new);
        l += w;
#pragma unroll
        for (int e = 0; e < E; ++e) o[e] = fmaf(w, g.v[r].get(e), o[e]);
    }
    m = m_new;
}

// E = d / 32 elements per lane (d in {32, 64, 128, 256}). A split is
// kAttWarps x kWarpRows rows; each warp prefetches its 64 row ids (2 per
// lane) once, then streams 8-row groups with the next group's K/V gathers in
// flight while the current group is reduced.
template <int E, typename KV>
__global__ void __launch_bounds__(kAttThreads) k4_sparse_attend(AttParams prm) {
    constexpr int D = 32 * E;
    __shared__ float s_m[kAttWarps], s_l[kAttWarps];
    __shared__ float s_o[kAttWarps][D];
    __shared__ uint32_t s_last;
    const uint32_t p = blockIdx.y, split = blockIdx.x;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

    const uint32_t c = prm.cnt[p];
    const uint32_t* list = prm.idx + (uint64_t)p * prm.idx_stride;
    uint32_t own;
    if (prm.partial_mode)
        own = prm.own_row ? prm.own_row[p] : kInv;
    else
        own = prm.n_valid[p / prm.nvalid_div] - 1u;
    const bool has_own = own != kInv;
    const bool own_listed = has_own && c > 0 && __ldg(list + c - 1) == own;
    const uint32_t nrows = c + ((has_own && !own_listed) ? 1u : 0u);

    const KV* kbase = static_cast<const KV*>(prm.kc) + (uint64_t)p * prm.stride_rows * D;
    const KV* vbase = static_cast<const KV*>(prm.vc) + (uint64_t)p * prm.stride_rows * D;

    const uint32_t wb = split * prm.rows_per_split + warp * kWarpRows;
    const uint32_t we = min(wb + kWarpRows, nrows);
    auto row_at = [&](uint32_t j) -> uint32_t {
        return j < we ? (j < c ? __ldg(list + j) : own) : kInv;
    };
    const uint32_t rid0 = row_at(wb + lane), rid1 = row_at(wb + 32 + lane);

    float qv[E];
#pragma unroll
    for (int e = 0; e < E; ++e) qv[e] = prm.q[(uint64_t)p * D + lane * E + e] * prm.qscale;
    float m = -INFINITY, l = 0.0f, o[E];
#pragma unroll
    for (int e = 0; e < E; ++e) o[e] = 0.0f;

    if (wb < we) {
        constexpr int G = Group<E, KV>::G;
        constexpr int PER_RID = 32 / G;  // groups per 32 prefetched ids
        const int ngroups = (int)((we - wb + G - 1) / G);
        Group<E, KV> ga, gb;
        ga.issue(rid0, 0, kbase, vbase, lane);
        for (int gi = 0; gi < ngroups; gi += 2) {
            const int g1 = gi + 1, g2 = gi + 2;
            if (g1 < ngroups) gb.issue(g1 < PER_RID ? rid0 : rid1, g1 % PER_RID, kbase, vbase, lane);
            consume(ga, qv, m, l, o);
            if (g1 >= ngroups) break;
            if (g2 < ngroups) ga.issue(g2 < PER_RID ? rid0 : rid1, g2 % PER_RID, kbase, vbase, lane);
            consume(gb, qv, m, l, o);
        }
    }

    // merge warps
    if (lane == 0) {
        s_m[warp] = m;
        s_l[warp] = l;
    }
#pragma unroll
    for (int e = 0; e < E; ++e) s_o[warp][lane * E + e] = o[e];
    __syncthreads();
    float M = -INFINITY;
#pragma unroll
    for (int w = 0; w < kAttWarps; ++w) M = fmaxf(M, s_m[w]);
    float* part = prm.partials + ((uint64_t)p * prm.nsplit + split) * (D + 2);
    for (int i = tid; i < D; i += kAttThreads) {
        float acc = 0.0f;
#pragma unroll
        for (int w = 0; w < kAttWarps; ++w)
            if (s_m[w] != -INFINITY) acc += s_o[w][i] * exp2f(s_m[w] - M);
        part[2 + i] = acc;
    }
    if (tid == 0) {
        float Ls = 0.0f;
#pragma unroll
        for (int w = 0; w < kAttWarps; ++w)
            if (s_m[w] != -INFINITY) Ls += s_l[w] * exp2f(s_m[w] - M);
        part[0] = M;
        part[1] = Ls;
    }

    // last split of this problem combines (K5)
    __threadfence();
    __syncthreads();
    if (tid == 0) {
        const uint32_t prev = atomicAdd(prm.counters + p, 1u);
        s_last = (prev + 1 == prm.nsplit) ? 1u : 0u;
    }
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    const float* parts = prm.partials + (uint64_t)p * prm.nsplit * (D + 2);
    float Mx = -INFINITY;
    for (uint32_t sidx = 0; sidx < prm.nsplit; ++sidx)
        Mx = fmaxf(Mx, __ldcg(parts + (uint64_t)sidx * (D + 2)));
    float Lx = 0.0f;
    for (uint32_t sidx = 0; sidx < prm.nsplit; ++sidx) {
        const float ms = __ldcg(parts + (uint64_t)sidx * (D + 2));
        if (ms != -INFINITY) Lx += __ldcg(parts + (uint64_t)sidx * (D + 2) + 1) * exp2f(ms - Mx);
    }
    for (int i = tid; i < D; i += kAttThreads) {
        float acc = 0.0f;
        for (uint32_t sidx = 0; sidx < prm.nsplit; ++sidx) {
            const float ms = __ldcg(parts + (uint64_t)sidx * (D + 2));
            if (ms != -INFINITY) acc += __ldcg(parts + (uint64_t)sidx * (D + 2) + 2 + i) * exp2f(ms - Mx);
        }
        if (prm.partial_mode)
            prm.out[(uint64_t)p * (D + 2) + 2 + i] = acc;
        else
            prm.out[(uint64_t)p * D + i] = acc / Lx;
    }
    if (tid == 0) {
        if (prm.partial_mode) {
            prm.out[(uint64_t)p * (D + 2)] = Mx;
            prm.out[(uint64_t)p * (D + 2) + 1] = Lx;
        }
        prm.counters[p] = 0u;
    }
}

// Merge R partial sets [R][P][d+2] (log2-domain m) -> out [P][d].
__global__ void k5_combine(const float* partials, uint32_t R, uint32_t P, uint32_t d,
                           float* out) {
    const uint32_t p = blockIdx.x;
    float M = -INFINITY;
    for (uint32_t r = 0; r < R; ++r) M = fmaxf(M, partials[((uint64_t)r * P + p) * (d + 2)]);
    float Ls = 0.0f;
    for (uint32_t r = 0; r < R; ++r) {
        const float* pr = partials + ((uint64_t)r * P + p) * (d + 2);
        if (pr[0] != -INFINITY) Ls += pr[1] * exp2f(pr[0] - M);
    }
    for (uint32_t i = threadIdx.x; i < d; i += blockDim.x) {
        float acc = 0.0f;
        for (uint32_t r = 0; r < R; ++r) {
            const float* pr = partials + ((uint64_t)r * P + p) * (d + 2);
            if (pr[0] != -INFINITY) acc += pr[2 + i] * exp2f(pr[0] - M);
        }
        out[(uint64_t)p * d + i] = acc / Ls;
    }
}

namespace {

template <int E>
const void* att_fn(int kv_dtype) {
    if (kv_dtype == SPL_BF16) return reinterpret_cast<const void*>(&k4_sparse_attend<E, __nv_bfloat16>);
    return reinterpret_cast<const void*>(&k4_sparse_attend<E, float>);
}

}  // namespace

spl_status sparse_attend_launch(spl_ctx* ctx, AttParams prm, uint32_t kmax, int kv_dtype,
                                cudaStream_t s) {
    const uint32_t d = prm.d;
    const void* fn = nullptr;
    switch (d) {
        case 32: fn = att_fn<1>(kv_dtype); break;
        case 64: fn = att_fn<2>(kv_dtype); break;
        case 128: fn = att_fn<4>(kv_dtype); break;
        case 256: fn = att_fn<8>(kv_dtype); break;
        default:
            return fail(ctx, SPL_E_DIMENSION,
                        "sparse_attend: head dim " + std::to_string(d) +
                            " not supported (32, 64, 128, 256)");
    }
    if (prm.P == 0) return SPL_OK;
    const uint64_t rows_max = (uint64_t)kmax + 1;
    const uint64_t R = (uint64_t)kAttWarps * kWarpRows;  // rows per split (CTA)
    const uint32_t nsplit = (uint32_t)((rows_max + R - 1) / R);
    prm.rows_per_split = (uint32_t)R;
    prm.nsplit = nsplit;
    const size_t part_bytes = (size_t)prm.P * nsplit * (d + 2) * sizeof(float);
    spl_status st = ensure_buffer(ctx, reinterpret_cast<void**>(&ctx->att_ws), &ctx->att_ws_bytes,
                                  part_bytes, false, s, "sparse_attend");
    if (st) return st;
    size_t have = ctx->att_counters_n * 4;
    st = ensure_buffer(ctx, reinterpret_cast<void**>(&ctx->att_counters), &have,
                       (size_t)prm.P * 4, true, s, "sparse_attend");
    if (st) return st;
    ctx->att_counters_n = have / 4;
    prm.partials = ctx->att_ws;
    prm.counters = ctx->att_counters;
    void* args[] = {&prm};
    SPL_CUDA_TRY(ctx, cudaLaunchKernel(fn, dim3(nsplit, prm.P), dim3(kAttThreads), args, 0, s));
    return after_launch(ctx, "k4_sparse_attend");
}

spl_status attend_combine_launch(spl_ctx* ctx, const float* partials, uint32_t R, uint32_t P,
                                 uint32_t d, float* out, cudaStream_t s) {
    if (P == 0) return SPL_OK;
    k5_combine<<<P, 128, 0, s>>>(partials, R, P, d, out);
    return after_launch(ctx, "k5_combine");
}

}  // namespace spl
