// K4/K5 — sparse decode attention over the retrieved rows (sm_100a).
//
// Replaces sparse_attention (attention_eval.cpp:234-264) + attend_subset
// (:54-78): per problem, softmax(q K_S^T * scale) V_S over S = picked U {own}
// (the own row n_valid - 1 is always attended, :249-260), fp32 accumulation.
//
// Flash-decoding split: a CTA (4 warps) takes 128 consecutive entries of the
// problem's row list; grid = splits x problems.
//   * logits, lane-per-row: lane i of a warp gathers its own K row with
//     16-byte loads (8 in flight) and dots it with q held in shared memory
//     (q pre-scaled by scale * log2(e): base-2 softmax), 4 partial sums —
//     no cross-lane reduction per row;
//   * warp softmax over its 32 rows (max / sum: 5 shuffles each);
//   * values, lane-per-dims: lane owns d/32 contiguous dims; for each row the
//     probability and row id are broadcast by shuffle and the V slice is one
//     coalesced 8 B (bf16) / 16 B (f32) load per lane, 8-16 rows in flight;
//   * warps merge (m, l, o) in shared memory; the CTA finishing a problem's
//     last split performs the log-sum-exp combine (K5) — one launch.
// Tolerance vs the reference (different summation order): max-abs 1e-5 with
// f32 K/V, 1e-3 with bf16 K/V (tests/test_gpu_parity.py).
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <string>

#include "spl_attend.cuh"
#include "spl_launch.cuh"

namespace spl {

constexpr int kAttThreads = 128;
constexpr int kAttWarps = kAttThreads / 32;
constexpr uint32_t kWarpRows = 32;  // one row per lane for the logits
constexpr uint32_t kInv = kAttInv;

// dot(q_s, K row) over D values, the row read as 16-byte chunks.
template <int D, typename KV>
__device__ __forceinline__ float row_dot(const KV* row, const float* q_s) {
    constexpr int NPER = 16 / (int)sizeof(KV);  // elements per 16-byte chunk
    constexpr int NCH = D / NPER;
    constexpr int BATCH = NCH < 8 ? NCH : 8;
    float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
    const uint4* p = reinterpret_cast<const uint4*>(row);
#pragma unroll
    for (int b0 = 0; b0 < NCH; b0 += BATCH) {
        uint4 v[BATCH];
#pragma unroll
        for (int i = 0; i < BATCH; ++i) v[i] = __ldg(p + b0 + i);
#pragma unroll
        for (int i = 0; i < BATCH; ++i) {
            const int e0 = (b0 + i) * NPER;
            const float4 qa = *reinterpret_cast<const float4*>(q_s + e0);
            if constexpr (sizeof(KV) == 2) {
                const float4 qb = *reinterpret_cast<const float4*>(q_s + e0 + 4);
                a0 = fmaf(qa.x, bf16lo(v[i].x), a0);
                a1 = fmaf(qa.y, bf16hi(v[i].x), a1);
                a2 = fmaf(qa.z, bf16lo(v[i].y), a2);
                a3 = fmaf(qa.w, bf16hi(v[i].y), a3);
                a0 = fmaf(qb.x, bf16lo(v[i].z), a0);
                a1 = fmaf(qb.y, bf16hi(v[i].z), a1);
                a2 = fmaf(qb.z, bf16lo(v[i].w), a2);
                a3 = fmaf(qb.w, bf16hi(v[i].w), a3);
            } else {
                a0 = fmaf(qa.x, __uint_as_float(v[i].x), a0);
                a1 = fmaf(qa.y, __uint_as_float(v[i].y), a1);
                a2 = fmaf(qa.z, __uint_as_float(v[i].z), a2);
                a3 = fmaf(qa.w, __uint_as_float(v[i].w), a3);
            }
        }
    }
    return (a0 + a1) + (a2 + a3);
}

__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Shared memory of a K4 CTA: per-warp (m, l, o) for the merge, the
// combine's per-split scales, the last-split flag.
template <int D>
struct AttSmem {
    float s_m[kAttWarps], s_l[kAttWarps];
    float s_o[kAttWarps][D];
    float s_cmb[2][kAttThreads];
    uint32_t s_last;
};

// End of a K4 CTA: merge the warps' (m, l, o) (lane-per-dims o: lane owns
// dims [lane*E, lane*E + E); l is the warp's total), then either write the
// result directly (one split) or write this split's partial and let the CTA
// finishing the problem's last split combine all of them (K5, log-sum-exp).
template <int E>
__device__ __forceinline__ void att_cta_finish(const AttParams& prm, AttSmem<32 * E>& sm,
                                               uint32_t p, uint32_t split, float m, float l,
                                               const float (&o)[E]) {
    constexpr int D = 32 * E;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    float* s_m = sm.s_m;
    float* s_l = sm.s_l;
    auto& s_o = sm.s_o;
    auto& s_cmb = sm.s_cmb;
    uint32_t& s_last = sm.s_last;
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
    if (prm.nsplit == 1) {
        // one split (short lists, e.g. config 1): the combine below reduces to
        // out = o / L with unit scales, so write the result directly (same
        // arithmetic) and skip the partials round trip and the counter
        float Ls = 0.0f;
#pragma unroll
        for (int w = 0; w < kAttWarps; ++w)
            if (s_m[w] != -INFINITY) Ls += s_l[w] * exp2f(s_m[w] - M);
        for (int i = tid; i < D; i += kAttThreads) {
            float acc = 0.0f;
#pragma unroll
            for (int w = 0; w < kAttWarps; ++w)
                if (s_m[w] != -INFINITY) acc += s_o[w][i] * exp2f(s_m[w] - M);
            if (prm.partial_mode)
                prm.out[(uint64_t)p * (D + 2) + 2 + i] = acc;
            else
                prm.out[(uint64_t)p * D + i] = acc / Ls;
        }
        if (tid == 0 && prm.partial_mode) {
            prm.out[(uint64_t)p * (D + 2)] = M;
            prm.out[(uint64_t)p * (D + 2) + 1] = Ls;
        }
        return;
    }
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
    // Combine in parallel: every (m, l) of the splits is fetched at once into
    // shared memory (one L2 round trip), the per-split scale factors computed
    // there, then each thread owns one output dim and streams the splits'
    // o[dim] with independent loads.
    const float* parts = prm.partials + (uint64_t)p * prm.nsplit * (D + 2);
    float Mx = -INFINITY, Lx = 0.0f;
    float acc[(D + kAttThreads - 1) / kAttThreads];
#pragma unroll
    for (int k = 0; k < (D + kAttThreads - 1) / kAttThreads; ++k) acc[k] = 0.0f;
    for (uint32_t s0 = 0; s0 < prm.nsplit; s0 += kAttThreads) {
        const uint32_t ns = min((uint32_t)kAttThreads, prm.nsplit - s0);
        float* s_scale = s_cmb[0];
        float* s_lv = s_cmb[1];
        __syncthreads();
        if ((uint32_t)tid < ns) {
            s_scale[tid] = __ldcg(parts + (uint64_t)(s0 + tid) * (D + 2));
            s_lv[tid] = __ldcg(parts + (uint64_t)(s0 + tid) * (D + 2) + 1);
        }
        __syncthreads();
        float Mc = -INFINITY;
        for (uint32_t i = 0; i < ns; ++i) Mc = fmaxf(Mc, s_scale[i]);
        const float Mn = fmaxf(Mx, Mc);
        const float rescale = Mx == -INFINITY ? 0.0f : exp2f(Mx - Mn);
        Lx *= rescale;
#pragma unroll
        for (int k = 0; k < (D + kAttThreads - 1) / kAttThreads; ++k) acc[k] *= rescale;
        Mx = Mn;
        __syncthreads();
        if ((uint32_t)tid < ns) {
            const float ms = s_scale[tid];
            s_scale[tid] = ms == -INFINITY ? 0.0f : exp2f(ms - Mx);
        }
        __syncthreads();
        for (uint32_t i = 0; i < ns; ++i) Lx += s_lv[i] * s_scale[i];
#pragma unroll
        for (int k = 0; k < (D + kAttThreads - 1) / kAttThreads; ++k) {
            const int dim = tid + k * kAttThreads;
            if (dim >= D) break;
            float a = 0.0f;
#pragma unroll 8
            for (uint32_t i = 0; i < ns; ++i)
                a = fmaf(__ldcg(parts + (uint64_t)(s0 + i) * (D + 2) + 2 + dim), s_scale[i], a);
            acc[k] += a;
        }
    }
#pragma unroll
    for (int k = 0; k < (D + kAttThreads - 1) / kAttThreads; ++k) {
        const int dim = tid + k * kAttThreads;
        if (dim >= D) break;
        if (prm.partial_mode)
            prm.out[(uint64_t)p * (D + 2) + 2 + dim] = acc[k];
        else
            prm.out[(uint64_t)p * D + dim] = acc[k] / Lx;
    }
    if (tid == 0) {
        if (prm.partial_mode) {
            prm.out[(uint64_t)p * (D + 2)] = Mx;
            prm.out[(uint64_t)p * (D + 2) + 1] = Lx;
        }
        prm.counters[p] = 0u;
    }
}

// Lane-per-row form (round 1; kept for A/B measurement, SPL_K4=lane): a
// warp takes 32 consecutive entries, lane i gathers row i's K with 16-byte
// loads, then the V rows lane-per-dims. E = d / 32 elements per lane.
template <int E, typename KV>
__global__ void __launch_bounds__(kAttThreads) k4_lane(AttParams prm) {
    constexpr int D = 32 * E;
    constexpr int VB = sizeof(KV) * E >= 16 ? 8 : 16;  // V rows in flight per lane
    __shared__ __align__(16) float q_s[D];
    __shared__ AttSmem<D> sm;
    const uint32_t p = blockIdx.y, split = blockIdx.x;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    pdl_trigger();
    pdl_wait();  // the row lists (and the appended own row) come from the previous kernels

    for (int i = tid; i < D; i += kAttThreads) q_s[i] = prm.q[(uint64_t)p * D + i] * prm.qscale;

    const uint32_t c = prm.cnt[p];
    const uint32_t* list = prm.idx + (uint64_t)p * prm.idx_stride;
    uint32_t own;
    if (prm.partial_mode && !prm.own_nvalid)
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
    const uint32_t nr = we > wb ? we - wb : 0;  // rows of this warp (warp-uniform)
    const uint32_t j = wb + lane;
    const uint32_t rid = j < we ? (j < c ? __ldg(list + j) : own) : kInv;
    __syncthreads();  // q_s

    float m = -INFINITY, l = 0.0f, o[E];
#pragma unroll
    for (int e = 0; e < E; ++e) o[e] = 0.0f;
    if (nr > 0) {
        // the V rows do not depend on the logits: start pulling this lane's V
        // row into L2 now so the value phase below does not pay a second
        // DRAM round trip after the K phase (random rows, cold L2)
        if (rid != kInv) {
            const char* vr = reinterpret_cast<const char*>(vbase + (uint64_t)rid * D);
#pragma unroll
            for (int b = 0; b < (int)(D * sizeof(KV)); b += 128)
                asm volatile("prefetch.global.L2 [%0];" ::"l"(vr + b));
        }
        float s = -INFINITY;
        if (rid != kInv) s = row_dot<D, KV>(kbase + (uint64_t)rid * D, q_s);
        m = warp_max(s);
        const float pr = rid != kInv ? exp2f(s - m) : 0.0f;
        l = warp_sum(pr);
        for (uint32_t r0 = 0; r0 < nr; r0 += VB) {
            VSlice<E, KV> vv[VB];
            float pw[VB];
#pragma unroll
            for (int i = 0; i < VB; ++i) {
                const uint32_t rr = __shfl_sync(0xffffffffu, rid, (r0 + i) & 31);
                pw[i] = __shfl_sync(0xffffffffu, pr, (r0 + i) & 31);
                if (r0 + i < nr) vv[i].load(vbase + (uint64_t)rr * D, lane);
            }
#pragma unroll
            for (int i = 0; i < VB; ++i) {
                if (r0 + i >= nr) break;
#pragma unroll
                for (int e = 0; e < E; ++e) o[e] = fmaf(pw[i], vv[i].get(e), o[e]);
            }
        }
    }

    att_cta_finish<E>(prm, sm, p, split, m, l, o);
}

// Warp-per-row gather form (the default): a warp takes RB x NB consecutive
// entries of the problem's row list and walks them in batches of RB = 8
// rows. For a batch, every lane issues its d/32-element slice of all 8 K rows
// AND all 8 V rows at once (the V rows do not depend on the logits), so one
// batch is one memory round trip with 16 coalesced row-slice loads in flight
// per lane (a warp reads each 256-byte bf16 row as one contiguous request);
// logits = rsum8 of the per-lane partial dots, online softmax in base 2 (q
// pre-scaled by scale * log2 e), o[lane's dims] += p_i * v_i. Measured on
// this B200 (tools/gather_sweep.cu): warp-per-row gathers of random 256-byte
// rows stream at the copy rate once enough are in flight, lane-per-row ones
// (k4_lane) do not.
template <int E, typename KV, int NB>
__global__ void __launch_bounds__(kAttThreads) k4_gather(AttParams prm) {
    constexpr int D = 32 * E;
    __shared__ AttSmem<D> sm;
    const uint32_t p = blockIdx.y, split = blockIdx.x;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    pdl_trigger();
    pdl_wait();

    const uint32_t c = prm.cnt[p];
    const uint32_t* list = prm.idx + (uint64_t)p * prm.idx_stride;
    uint32_t own;
    if (prm.partial_mode && !prm.own_nvalid)
        own = prm.own_row ? prm.own_row[p] : kInv;
    else
        own = prm.n_valid[p / prm.nvalid_div] - 1u;
    const bool has_own = own != kInv;
    const bool own_listed = has_own && c > 0 && __ldg(list + c - 1) == own;
    const uint32_t nrows = c + ((has_own && !own_listed) ? 1u : 0u);
    const KV* kbase = static_cast<const KV*>(prm.kc) + (uint64_t)p * prm.stride_rows * D;
    const KV* vbase = static_cast<const KV*>(prm.vc) + (uint64_t)p * prm.stride_rows * D;
    // this lane's slice of q, pre-scaled
    float qv[E];
#pragma unroll
    for (int e = 0; e < E; ++e) qv[e] = __ldg(prm.q + (uint64_t)p * D + lane * E + e) * prm.qscale;

    constexpr uint32_t kWR = kAttRB * NB;  // entries per warp (<= 32)
    static_assert(kWR <= 32, "one row id per lane");
    const uint32_t wb = split * prm.rows_per_split + warp * kWR;
    const uint32_t we = min(wb + kWR, nrows);
    float m = -INFINITY, lsum = 0.0f, o[E];
#pragma unroll
    for (int e = 0; e < E; ++e) o[e] = 0.0f;
    if (wb < we) warp_attend<E, KV>(kbase, vbase, list, c, own, wb, we, qv, m, lsum, o);
    const float l = attend_lsum_total(lsum);
    att_cta_finish<E>(prm, sm, p, split, m, l, o);
}

// Any head dim (the reference's API accepts every d; the tuned kernel above
// covers d in {32, 64, 128, 256}). One warp per problem, rows processed one
// at a time with a warp-reduced dot product; f32 only (the drop-in API feeds
// f32 K/V). Same log-sum-exp semantics; partial mode supported.
__global__ void k4_attend_generic(AttParams prm) {
    const uint32_t p = blockIdx.x;
    const int lane = threadIdx.x;
    const uint32_t d = prm.d;
    const uint32_t c = prm.cnt[p];
    const uint32_t* list = prm.idx + (uint64_t)p * prm.idx_stride;
    uint32_t own;
    if (prm.partial_mode && !prm.own_nvalid)
        own = prm.own_row ? prm.own_row[p] : kInv;
    else
        own = prm.n_valid[p / prm.nvalid_div] - 1u;
    const bool has_own = own != kInv;
    const bool own_listed = has_own && c > 0 && list[c - 1] == own;
    const uint32_t nrows = c + ((has_own && !own_listed) ? 1u : 0u);
    const float* K = static_cast<const float*>(prm.kc) + (uint64_t)p * prm.stride_rows * d;
    const float* V = static_cast<const float*>(prm.vc) + (uint64_t)p * prm.stride_rows * d;
    const float* q = prm.q + (uint64_t)p * d;
    float m = -INFINITY, l = 0.0f;
    float* o = prm.partials + (uint64_t)p * d;  // scratch accumulator [P][d]
    for (uint32_t i = lane; i < d; i += 32) o[i] = 0.0f;
    for (uint32_t j = 0; j < nrows; ++j) {
        const uint32_t r = j < c ? list[j] : own;
        float part = 0.0f;
        for (uint32_t i = lane; i < d; i += 32) part = fmaf(q[i] * prm.qscale, K[(uint64_t)r * d + i], part);
        const float s = warp_sum(part);
        const float mn = fmaxf(m, s);
        const float corr = exp2f(m - mn), w = exp2f(s - mn);
        l = l * corr + w;
        for (uint32_t i = lane; i < d; i += 32) o[i] = o[i] * corr + w * V[(uint64_t)r * d + i];
        m = mn;
    }
    for (uint32_t i = lane; i < d; i += 32) {
        if (prm.partial_mode)
            prm.out[(uint64_t)p * (d + 2) + 2 + i] = o[i];
        else
            prm.out[(uint64_t)p * d + i] = o[i] / l;
    }
    if (prm.partial_mode && lane == 0) {
        prm.out[(uint64_t)p * (d + 2)] = m;
        prm.out[(uint64_t)p * (d + 2) + 1] = l;
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

// SPL_K4=lane selects the round-1 lane-per-row kernel (A/B measurements);
// SPL_K4_NB=1|2|4 the batches per warp of the gather kernel (default 4).
int k4_mode() {
    static const int m = [] {
        const char* e = getenv("SPL_K4");
        return (e && e[0] == 'l') ? 1 : 0;
    }();
    return m;
}
int k4_nb() {
    static const int nb = [] {
        const char* e = getenv("SPL_K4_NB");
        const int v = e ? atoi(e) : 0;
        return (v == 1 || v == 2 || v == 4) ? v : 4;  // 4: config-4 step 590 -> 570 us
    }();
    return nb;
}
template <int E, typename KV>
const void* gather_fn(int nb) {
    if (nb == 1) return reinterpret_cast<const void*>(&k4_gather<E, KV, 1>);
    if (nb == 4) return reinterpret_cast<const void*>(&k4_gather<E, KV, 4>);
    return reinterpret_cast<const void*>(&k4_gather<E, KV, 2>);
}
template <int E>
const void* att_fn(int kv_dtype) {
    if (k4_mode() == 1) {
        if (kv_dtype == SPL_BF16) return reinterpret_cast<const void*>(&k4_lane<E, __nv_bfloat16>);
        return reinterpret_cast<const void*>(&k4_lane<E, float>);
    }
    if (kv_dtype == SPL_BF16) return gather_fn<E, __nv_bfloat16>(k4_nb());
    return gather_fn<E, float>(k4_nb());
}

}  // namespace

// Size K4's workspace (partials + counters) for P problems of up to kmax
// listed rows and head dim d, before any launch of a call that must not
// allocate between its kernels (the sharded step: an allocation or a
// zero-fill synchronisation while a kernel of the step waits for its peers
// would stall it).
spl_status sparse_attend_reserve(spl_ctx* ctx, uint32_t P, uint32_t kmax, uint32_t d, cudaStream_t s) {
    const uint64_t R = att_rows_per_split();
    const uint64_t nsplit = ((uint64_t)kmax + 1 + R - 1) / R;
    const size_t dd = d > 128 ? d : 128;  // the fused decode step's partials use d = 128 too
    spl_status st = ensure_buffer(ctx, reinterpret_cast<void**>(&ctx->att_ws), &ctx->att_ws_bytes,
                                  (size_t)P * nsplit * (dd + 2) * sizeof(float), false, s,
                                  "sparse_attend");
    if (st) return st;
    size_t have = ctx->att_counters_n * 4;
    st = ensure_buffer(ctx, reinterpret_cast<void**>(&ctx->att_counters), &have, (size_t)P * 4, true,
                       s, "sparse_attend");
    if (st) return st;
    ctx->att_counters_n = have / 4;
    return SPL_OK;
}

uint32_t att_rows_per_split() {
    return k4_mode() == 1 ? (uint32_t)(kAttWarps * kWarpRows) : (uint32_t)(kAttWarps * kAttRB * k4_nb());
}

spl_status sparse_attend_launch(spl_ctx* ctx, AttParams prm, uint32_t kmax, int kv_dtype,
                                cudaStream_t s) {
    const uint32_t d = prm.d;
    const void* fn = nullptr;
    if (kv_dtype != SPL_F32 && kv_dtype != SPL_BF16)
        return fail(ctx, SPL_E_DIMENSION, "sparse_attend: unknown kv dtype");
    // the tuned kernels read K / V row slices with 8- / 16-byte loads: caches
    // that are not 16-byte aligned take the generic kernel (f32) or fail
    const bool aligned =
        ((reinterpret_cast<uintptr_t>(prm.kc) | reinterpret_cast<uintptr_t>(prm.vc)) & 15u) == 0;
    if (!aligned && kv_dtype == SPL_BF16 && (d == 32 || d == 64 || d == 128 || d == 256))
        return fail(ctx, SPL_E_DIMENSION, "sparse_attend: bf16 K / V caches must be 16-byte aligned");
    switch (aligned ? d : 0u) {
        case 32: fn = att_fn<1>(kv_dtype); break;
        case 64: fn = att_fn<2>(kv_dtype); break;
        case 128: fn = att_fn<4>(kv_dtype); break;
        case 256: fn = att_fn<8>(kv_dtype); break;
        default: {
            if (prm.d == 0) return fail(ctx, SPL_E_DIMENSION, "attention: embedding dimensions differ");
            if (kv_dtype != SPL_F32)
                return fail(ctx, SPL_E_DIMENSION,
                            "sparse_attend: bf16 K/V needs head dim 32, 64, 128 or 256");
            if (prm.P == 0) return SPL_OK;
            spl_status st = ensure_buffer(ctx, reinterpret_cast<void**>(&ctx->att_ws),
                                          &ctx->att_ws_bytes, (size_t)prm.P * d * sizeof(float),
                                          false, s, "sparse_attend");
            if (st) return st;
            prm.partials = ctx->att_ws;
            k4_attend_generic<<<prm.P, 32, 0, s>>>(prm);
            return after_launch(ctx, "k4_attend_generic");
        }
    }
    if (prm.P == 0) return SPL_OK;
    const uint64_t rows_max = (uint64_t)kmax + 1;
    const uint64_t R = att_rows_per_split();  // rows per split (CTA)
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
    SPL_CUDA_TRY(ctx, launch_pdl(fn, dim3(nsplit, prm.P), dim3(kAttThreads), 0, s, args));
    return after_launch(ctx, k4_mode() == 1 ? "k4_lane" : "k4_gather");
}

spl_status attend_combine_launch(spl_ctx* ctx, const float* partials, uint32_t R, uint32_t P,
                                 uint32_t d, float* out, cudaStream_t s) {
    if (P == 0) return SPL_OK;
    k5_combine<<<P, 128, 0, s>>>(partials, R, P, d, out);
    return after_launch(ctx, "k5_combine");
}

// Force the lazy load of every K4 variant (see encode_preload).
void attend_preload() {
    cudaFuncAttributes a;
    const void* fns[] = {att_fn<1>(SPL_BF16), att_fn<1>(SPL_F32), att_fn<2>(SPL_BF16),
                         att_fn<2>(SPL_F32),  att_fn<4>(SPL_BF16), att_fn<4>(SPL_F32),
                         att_fn<8>(SPL_BF16), att_fn<8>(SPL_F32),
                         reinterpret_cast<const void*>(&k4_attend_generic),
                         reinterpret_cast<const void*>(&k5_combine)};
    for (const void* f : fns) cudaFuncGetAttributes(&a, f);
}

}  // namespace spl
