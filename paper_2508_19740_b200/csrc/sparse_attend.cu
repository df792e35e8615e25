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

template <int E, typename KV>
struct RowVec;
template <int E>
struct RowVec<E, __nv_bfloat16> {
    float f[E];
    __device__ __forceinline__ void load(const __nv_bfloat16* row, int lane) {
        const __nv_bfloat16* p = row + lane * E;
        if constexpr (E == 4) {
            const uint2 u = __ldg(reinterpret_cast<const uint2*>(p));
            const __nv_bfloat162 a = *reinterpret_cast<const __nv_bfloat162*>(&u.x);
            const __nv_bfloat162 b = *reinterpret_cast<const __nv_bfloat162*>(&u.y);
            f[0] = __low2float(a); f[1] = __high2float(a);
            f[2] = __low2float(b); f[3] = __high2float(b);
        } else if constexpr (E == 8) {
            const uint4 u = __ldg(reinterpret_cast<const uint4*>(p));
            const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const __nv_bfloat162 t = *reinterpret_cast<const __nv_bfloat162*>(&w[i]);
                f[2 * i] = __low2float(t);
                f[2 * i + 1] = __high2float(t);
            }
        } else if constexpr (E == 2) {
            const __nv_bfloat162 t = __ldg(reinterpret_cast<const __nv_bfloat162*>(p));
            f[0] = __low2float(t); f[1] = __high2float(t);
        } else {
#pragma unroll
            for (int i = 0; i < E; ++i) f[i] = __bfloat162float(p[i]);
        }
    }
};
template <int E>
struct RowVec<E, float> {
    float f[E];
    __device__ __forceinline__ void load(const float* row, int lane) {
        const float* p = row + lane * E;
        if constexpr (E % 4 == 0) {
#pragma unroll
            for (int i = 0; i < E; i += 4) {
                const float4 u = __ldg(reinterpret_cast<const float4*>(p + i));
                f[i] = u.x; f[i + 1] = u.y; f[i + 2] = u.z; f[i + 3] = u.w;
            }
        } else if constexpr (E == 2) {
            const float2 u = __ldg(reinterpret_cast<const float2*>(p));
            f[0] = u.x; f[1] = u.y;
        } else {
#pragma unroll
            for (int i = 0; i < E; ++i) f[i] = __ldg(p + i);
        }
    }
};

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// E = d / 32 elements per lane (d in {32, 64, 128, 256}).
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
        own = prm.own_row ? prm.own_row[p] : 0xFFFFFFFFu;
    else
        own = prm.n_valid[p / prm.nvalid_div] - 1u;
    const bool has_own = own != 0xFFFFFFFFu;
    const bool own_listed = has_own && c > 0 && __ldg(list + c - 1) == own;
    const uint32_t nrows = c + ((has_own && !own_listed) ? 1u : 0u);
    const uint32_t start = split * prm.rows_per_split;
    const uint32_t end = min(start + prm.rows_per_split, nrows);

    const KV* kbase = static_cast<const KV*>(prm.kc) + (uint64_t)p * prm.stride_rows * D;
    const KV* vbase = static_cast<const KV*>(prm.vc) + (uint64_t)p * prm.stride_rows * D;
    float qv[E];
#pragma unroll
    for (int e = 0; e < E; ++e) qv[e] = prm.q[(uint64_t)p * D + lane * E + e] * prm.qscale;

    float m = -INFINITY, l = 0.0f, o[E];
#pragma unroll
    for (int e = 0; e < E; ++e) o[e] = 0.0f;

    // warp w takes a contiguous chunk of this split's rows
    const uint32_t span = end > start ? end - start : 0;
    const uint32_t chunk = (span + kAttWarps - 1) / kAttWarps;
    const uint32_t wb = start + min(span, chunk * warp), we = start + min(span, chunk * (warp + 1));
    for (uint32_t j = wb; j < we; j += kGroup) {
        // lanes 0..7 fetch the group's row ids
        uint32_t rid = 0xFFFFFFFFu;
        if (lane < kGroup && j + lane < we) rid = (j + lane < c) ? __ldg(list + j + lane) : own;
        RowVec<E, KV> kr[kGroup], vr[kGroup];
        uint32_t rows[kGroup];
#pragma unroll
        for (int r = 0; r < kGroup; ++r) {
            rows[r] = __shfl_sync(0xffffffffu, rid, r);
            if (rows[r] != 0xFFFFFFFFu) {
                kr[r].load(kbase + (uint64_t)rows[r] * D, lane);
                vr[r].load(vbase + (uint64_t)rows[r] * D, lane);
            }
        }
        float s[kGroup];
        float gmax = -INFINITY;
#pragma unroll
        for (int r = 0; r < kGroup; ++r) {
            float part = 0.0f;
            if (rows[r] != 0xFFFFFFFFu) {
#pragma unroll
                for (int e = 0; e < E; ++e) part = fmaf(qv[e], kr[r].f[e], part);
            }
            part = warp_sum(part);
            s[r] = rows[r] != 0xFFFFFFFFu ? part : -INFINITY;
            gmax = fmaxf(gmax, s[r]);
        }
        const float m_new = fmaxf(m, gmax);
        const float corr = exp2f(m - m_new);  // m = -inf -> 0
        l *= corr;
#pragma unroll
        for (int e = 0; e < E; ++e) o[e] *= corr;
#pragma unroll
        for (int r = 0; r < kGroup; ++r) {
            if (rows[r] == 0xFFFFFFFFu) continue;
            const float w = exp2f(s[r] - m_new);
            l += w;
#pragma unroll
            for (int e = 0; e < E; ++e) o[e] = fmaf(w, vr[r].f[e], o[e]);
        }
        m = m_new;
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
    // enough CTAs to cover every SM several times, >= 32 rows per warp-group
    const uint64_t target_ctas = (uint64_t)ctx->num_sms * 8;
    uint64_t R = (rows_max * prm.P + target_ctas - 1) / target_ctas;
    R = std::max<uint64_t>(64, std::min<uint64_t>(1024, (R + 31) / 32 * 32));
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
