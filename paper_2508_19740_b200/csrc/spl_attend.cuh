// Warp-level sparse-attention building blocks shared by K4 (sparse_attend.cu)
// and the decode-step form of K3 that attends the rows it selects
// (hamming_topk.cu, k3_fused<.., ATT>). Semantics of attend_subset
// (attention_eval.cpp:54-78): logits q.k * scale, max, w = exp(l - max),
// out = sum w v / sum w — here in base 2 (q pre-scaled by scale * log2 e),
// online over batches, fp32 accumulation.
#pragma once
#include <cuda_bf16.h>
#include <stdint.h>

namespace spl {

constexpr uint32_t kAttInv = 0xFFFFFFFFu;  // "no row"
constexpr int kAttRB = 8;                   // rows per warp batch

__device__ __forceinline__ float bf16lo(uint32_t w) { return __uint_as_float(w << 16); }
__device__ __forceinline__ float bf16hi(uint32_t w) { return __uint_as_float(w & 0xffff0000u); }

// A lane's E-element slice [lane*E, lane*E + E) of a K or V row.
template <int E, typename KV>
struct VSlice;
template <int E>
struct VSlice<E, __nv_bfloat16> {
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
    __device__ __forceinline__ void zero() {
#pragma unroll
        for (int i = 0; i < (E + 1) / 2; ++i) u[i] = 0u;
    }
    __device__ __forceinline__ float get(int e) const {
        return (e & 1) ? bf16hi(u[e / 2]) : bf16lo(u[e / 2]);
    }
};
template <int E>
struct VSlice<E, float> {
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
    __device__ __forceinline__ void zero() {
#pragma unroll
        for (int i = 0; i < E; ++i) f[i] = 0.0f;
    }
    __device__ __forceinline__ float get(int e) const { return f[e]; }
};

// Sum of eight per-lane partial values over the warp with 9 shuffles
// instead of 8 x 5: three halving exchanges (xor 16, 8, 4) leave lane l with
// row r(l) = 4*b4 + 2*b3 + b2 (b = bits of l) summed over 8 lanes, then xor 2
// and xor 1 finish it. Every lane returns the full sum of its row r(l).
__device__ __forceinline__ uint32_t rsum8_row(int lane) {
    return ((lane >> 4) & 1) * 4 + ((lane >> 3) & 1) * 2 + ((lane >> 2) & 1);
}
__device__ __forceinline__ int rsum8_lane(int row) {
    return ((row >> 2) << 4) | (((row >> 1) & 1) << 3) | ((row & 1) << 2);
}
__device__ __forceinline__ float rsum8(const float (&x)[8], int lane) {
    const bool b4 = (lane >> 4) & 1, b3 = (lane >> 3) & 1, b2 = (lane >> 2) & 1;
    float t[4], u[2];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const float mine = b4 ? x[j + 4] : x[j], other = b4 ? x[j] : x[j + 4];
        t[j] = mine + __shfl_xor_sync(0xffffffffu, other, 16);
    }
#pragma unroll
    for (int j = 0; j < 2; ++j) {
        const float mine = b3 ? t[j + 2] : t[j], other = b3 ? t[j] : t[j + 2];
        u[j] = mine + __shfl_xor_sync(0xffffffffu, other, 8);
    }
    float v = (b2 ? u[1] : u[0]) + __shfl_xor_sync(0xffffffffu, b2 ? u[0] : u[1], 4);
    v += __shfl_xor_sync(0xffffffffu, v, 2);
    v += __shfl_xor_sync(0xffffffffu, v, 1);
    return v;
}

// One online-softmax step over a loaded 8-row batch (see warp_attend).
template <int E, typename KV>
__device__ __forceinline__ void attend_batch8(const VSlice<E, KV> (&kk)[kAttRB],
                                              const VSlice<E, KV> (&vv)[kAttRB], bool my_valid,
                                              int lane, const float (&qv)[E], float& m,
                                              float& lsum, float (&o)[E]) {
    float part[kAttRB];
#pragma unroll
    for (int i = 0; i < kAttRB; ++i) {
        float a = 0.0f;
#pragma unroll
        for (int e = 0; e < E; ++e) a = fmaf(qv[e], kk[i].get(e), a);
        part[i] = a;
    }
    float s = rsum8(part, lane);
    if (!my_valid) s = -INFINITY;
    float mb = fmaxf(s, __shfl_xor_sync(0xffffffffu, s, 4));
    mb = fmaxf(mb, __shfl_xor_sync(0xffffffffu, mb, 8));
    mb = fmaxf(mb, __shfl_xor_sync(0xffffffffu, mb, 16));
    const float mn = fmaxf(m, mb);  // finite: the batch has a valid row
    const float corr = exp2f(m - mn);
    const float pr = exp2f(s - mn);  // 0 for "no row"
    lsum = lsum * corr + pr;
#pragma unroll
    for (int e = 0; e < E; ++e) o[e] *= corr;
#pragma unroll
    for (int i = 0; i < kAttRB; ++i) {
        const float pi = __shfl_sync(0xffffffffu, pr, rsum8_lane(i));
#pragma unroll
        for (int e = 0; e < E; ++e) o[e] = fmaf(pi, vv[i].get(e), o[e]);
    }
    m = mn;
}

// One warp attends entries [j0, j1) of a row list: entry j is ids[j] for
// j < nlist, `extra` for j == nlist (the own row when it is not listed).
// Warp-per-row gather: per batch of 8 rows every lane issues its slice of all
// 8 K rows AND all 8 V rows at once (V does not depend on the logits), so a
// batch is one memory round trip with 16 row-slice loads in flight per lane
// and each 256-byte bf16 row read as one contiguous warp request; row ids
// are fetched 32 at a time (one per lane; IDS_SMEM: ids is shared memory). Online softmax: (m, lsum, o)
// carry across calls; lsum is per lane for its rsum8 row (4 lanes per row),
// reduce it with attend_lsum_total at the end. qv = this lane's slice of q
// already scaled by scale * log2(e).
// The lane's own-row validity comes from a shuffle of the id (not from an
// array indexed by the lane's rsum8 row, which the compiler kept in local
// memory): no spills in the decode-step kernel, config-2 step ~1 us faster.
template <int E, typename KV, bool IDS_SMEM = false>
__device__ __forceinline__ void warp_attend(const KV* kbase, const KV* vbase, const uint32_t* ids,
                                            uint32_t nlist, uint32_t extra, uint32_t j0,
                                            uint32_t j1, const float (&qv)[E], float& m,
                                            float& lsum, float (&o)[E]) {
    constexpr int D = 32 * E;
    const int lane = threadIdx.x & 31;
    const uint32_t myrow = rsum8_row(lane);
    for (uint32_t jb = j0; jb < j1; jb += 32) {
        const uint32_t j = jb + lane;
        const uint32_t myid =
            j < j1 ? (j < nlist ? (IDS_SMEM ? ids[j] : __ldcg(ids + j)) : extra) : kAttInv;
#pragma unroll 1
        for (int b = 0; b < 4; ++b) {
            if (jb + b * kAttRB >= j1) break;  // warp-uniform
            VSlice<E, KV> kk[kAttRB], vv[kAttRB];
#pragma unroll
            for (int i = 0; i < kAttRB; ++i) {
                const uint32_t rid = __shfl_sync(0xffffffffu, myid, b * kAttRB + i);
                if (rid != kAttInv) {
                    kk[i].load(kbase + (uint64_t)rid * D, lane);
                    vv[i].load(vbase + (uint64_t)rid * D, lane);
                } else {
                    kk[i].zero();
                    vv[i].zero();
                }
            }
            const bool my_valid = __shfl_sync(0xffffffffu, myid, b * kAttRB + (int)myrow) != kAttInv;
            attend_batch8<E, KV>(kk, vv, my_valid, lane, qv, m, lsum, o);
        }
    }
}

// Total of the per-lane lsum of warp_attend: the 8 row groups are the lanes
// that differ in bits 2..4.
__device__ __forceinline__ float attend_lsum_total(float lsum) {
    float l = lsum + __shfl_xor_sync(0xffffffffu, lsum, 4);
    l += __shfl_xor_sync(0xffffffffu, l, 8);
    l += __shfl_xor_sync(0xffffffffu, l, 16);
    return l;
}

}  // namespace spl
