// Threshold / tie-quota arithmetic of the bit-exact top-k select, shared by
// the device planner and the host (spl_plan_shard_host, CPU tests).
//
// The reference keeps the k entries that rank ahead under (score desc, index
// asc) (bitcodes.cpp:97-103). With integer scores in [0, L] that set is
// exactly: every row with score > T, plus the FIRST `quota` rows (lowest
// index) with score == T, where T = max{t : #(score >= t) >= k} and
// quota = k - #(score > T). When rows are split into contiguous, ordered
// pieces (CTA segments on one GPU, ranks of a sequence-sharded cache), piece
// j takes min(eq_j, max(0, quota - eq_before_j)) of its ties, and its first
// output lands at gt_before_j + min(eq_before_j, quota).
#pragma once
#include <stdint.h>

#if defined(__CUDACC__)
#define SPL_PLAN_HD __host__ __device__ __forceinline__
#else
#define SPL_PLAN_HD static inline
#endif

#define SPL_PLAN_SKIP 0xFFFFFFFFu

struct spl_shard_plan {
    uint32_t T;       // threshold score (SPL_PLAN_SKIP when nothing is selected)
    uint32_t quota;   // global number of ties (score == T) to keep
    uint32_t take_eq; // ties kept by this piece
    uint32_t count;   // indices emitted by this piece
    uint32_t offset;  // position of this piece's first index in the global list
    uint32_t kk;      // global budget min(k, total valid)
};

// hist: R rows of L+1 counts, row r at hist + r * rank_stride.
SPL_PLAN_HD spl_shard_plan spl_plan_shard(const uint32_t* hist, uint64_t rank_stride,
                                          uint32_t R, uint32_t rank, uint32_t L, uint32_t k) {
    spl_shard_plan out = {SPL_PLAN_SKIP, 0, 0, 0, 0, 0};
    uint64_t n = 0;
    for (uint32_t r = 0; r < R; ++r)
        for (uint32_t t = 0; t <= L; ++t) n += hist[r * rank_stride + t];
    const uint64_t kk = k < n ? k : n;
    out.kk = (uint32_t)kk;
    if (kk == 0) return out;
    uint64_t ge = 0;  // #(score > t) while descending
    uint32_t T = 0;
    uint64_t gt_total = 0;
    for (int64_t t = L; t >= 0; --t) {
        uint64_t at = 0;
        for (uint32_t r = 0; r < R; ++r) at += hist[r * rank_stride + (uint32_t)t];
        if (ge + at >= kk) {
            T = (uint32_t)t;
            gt_total = ge;
            break;
        }
        ge += at;
    }
    const uint64_t quota = kk - gt_total;
    uint64_t eq_before = 0, gt_before = 0;
    for (uint32_t r = 0; r < rank; ++r) {
        eq_before += hist[r * rank_stride + T];
        for (uint32_t t = T + 1; t <= L; ++t) gt_before += hist[r * rank_stride + t];
    }
    const uint64_t eq_mine = hist[(uint64_t)rank * rank_stride + T];
    uint64_t gt_mine = 0;
    for (uint32_t t = T + 1; t <= L; ++t) gt_mine += hist[(uint64_t)rank * rank_stride + t];
    const uint64_t left = quota > eq_before ? quota - eq_before : 0;
    const uint64_t take = eq_mine < left ? eq_mine : left;
    out.T = T;
    out.quota = (uint32_t)quota;
    out.take_eq = (uint32_t)take;
    out.count = (uint32_t)(gt_mine + take);
    out.offset = (uint32_t)(gt_before + (eq_before < quota ? eq_before : quota));
    return out;
}
