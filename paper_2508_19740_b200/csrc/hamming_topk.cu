// K3 — HBM-streaming Hamming scan + bit-exact top-k select (sm_100a).
//
// Replaces nxor_scores_into (bitcodes.cpp:59-76) + top_k_indices<int32_t>
// (bitcodes.cpp:89-131) as hash_topk composes them (attention_eval.cpp:
// 172-179), batched over P (batch, head) problems.
//
// Layout: codes [P][stride][W] u32 (row = one 16 B / 32 B vector for
// L = 128 / 256). The virtual row space P x n_max is cut into G equal
// contiguous CTA ranges (G = SMs x resident CTAs: exactly one wave); a CTA's
// range is split at problem boundaries into "segments" (record index
// cta + problem, unique because the (cta, problem) staircase is monotone).
//
// Streaming: every thread keeps two sets of U 32-byte units in flight
// (LDG.E.NA.EFL2.256: 256-bit, no L1 allocation, L2 evict-first; register
// double buffering), score = L - sum popc(q ^ r), and counts scores in
// per-thread private u8 counters in shared memory (LDS/STS, conflict-free,
// flushed into a u32 histogram before they can wrap) — a shared-atomic
// histogram cannot keep up with ~1.5 rows/clk/SM.
//
// Fused path (k3_fused, see below): when the scores fit in shared memory (the
// headline 32 x 512K case), one plain launch streams, histograms,
// derives T / tie quota / offsets and compacts from shared memory, with
// per-problem readiness waits only. One launch, one HBM pass.
// Two-pass path (k3_scan + k3_select): u8/u16 scores to an L2-resident
// buffer; the CTA finishing a problem's last segment plans it; k3_select
// compacts. Used for caches too large for on-chip scores and for the
// sequence-sharded (multi-GPU) flow, whose plan needs a collective between
// the two kernels.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cstdio>
#include <string>
#include <vector>
#include <cstring>

#include "spl_attend.cuh"
#include "spl_launch.cuh"
#include "spl_plan.cuh"

namespace spl {

struct K3Geom {
    uint64_t n_max;    // rows per problem (cache capacity; rows >= n_max are never scored)
    uint64_t pstride;  // rows per problem in the virtual row space (>= n_max; the fused
                       // plan pads it to whole segments so no CTA straddles two problems)
    uint64_t total;    // P * pstride
    uint64_t S;      // rows per CTA
    uint64_t n_pad;  // global score row stride (two-pass)
    uint32_t G;      // CTAs
    uint32_t P;
};

__host__ __device__ __forceinline__ uint32_t seg_first(const K3Geom& g, uint32_t p) {
    return (uint32_t)(((uint64_t)p * g.pstride) / g.S);
}
__host__ __device__ __forceinline__ uint32_t seg_last(const K3Geom& g, uint32_t p) {
    return (uint32_t)((((uint64_t)p + 1) * g.pstride - 1) / g.S);
}

struct K3Params {
    const uint32_t* codes;
    uint64_t stride_rows;
    const uint32_t* qcodes;
    const uint32_t* n_valid;
    uint32_t nvalid_div;
    uint32_t L;
    uint32_t W;
    uint32_t k;
    K3Geom g;
    void* scores;          // two-pass: [P][n_pad] ScoreT
    uint32_t* records;     // [(G+P)][L+2] suffix-cumulative counts
    uint32_t* tot_hist;    // [P][tot_stride] per-problem histogram (atomics)
    uint64_t tot_stride;
    uint32_t* counters;    // [P] two-pass segment completion
    uint32_t* sync;        // [2] fused: grid barrier, completion
    uint4* plans;          // [(G+P)] two-pass {T, offset, take, 0}
    uint32_t* cnt_out;     // [P]
    uint32_t* idx_out;     // fused: [P][idx_stride]
    uint64_t idx_stride;
    uint32_t* dev_err;
    int shard;             // 1: no planning; tot_hist = caller's histogram
    uint32_t score_region; // fused: bytes of shared memory for scores
    uint64_t* trace;       // optional [G][8] globaltimer stamps (SPL_K3_TRACE)
    uint32_t hist_lo;      // fused: private counters cover scores [hist_lo, L] only
    uint32_t* counters2;   // fused: [P] low-bin fallback completion
    int clamp8;            // two-pass L = 256: u8 scores hold min(score, 255)
    // fused sequence-sharded path (k3_fused<.., SHARD = true>): per-problem
    // histograms are exchanged with the other ranks inside the kernel through
    // their exchange areas (IPC-mapped peer memory over NVLink)
    uint32_t** peer_bufs;  // [R] exchange area of every rank (own included)
    uint32_t* own_buf;     // this rank's exchange area
    uint32_t R, rank, Pmax;
    uint32_t* epoch_ptr;   // the group's call counter (device; advanced by the last CTA)
    uint32_t* out_offset;  // [P] position of this rank's first index in the global list
    // optional (decode step): K / V caches laid out like the codes ([P][stride_rows]
    // rows of pf_row_bytes); the fused select prefetches every emitted row of
    // both into L2 so the attention gather that follows finds them there
    const char* pf_k;
    const char* pf_v;
    uint32_t pf_row_bytes;
    // decode step (k3_fused<.., ATT>): every CTA attends the rows it just
    // selected (K/V rows at pf_k / pf_v, head dim 128) and the CTA finishing a
    // problem's last segment combines the per-segment partials (log-sum-exp)
    const float* att_q;    // [P][128] f32 queries
    float att_qscale;      // scale * log2(e)
    float* att_part;       // [(G + P)][130] per-segment (m, l, o[128])
    uint32_t* att_cnt;     // [P] segments attended (self-resetting)
    float* att_out;        // [P][128]
    int att_own;           // this rank holds the own row (n_valid - 1): always 1
                           // unsharded; sharded decode: the rank the new token went to
    uint32_t part_off;     // sharded decode: u32 offset of the partial-exchange area in
                           // every rank's peer buffer (after the histogram area)
};

constexpr int kThreads = 256;
// Shared memory per SM the fused plan may use: above this the driver must
// pick the 228 KB carve-out (L1 ~0), and streaming LDG.256 reads drop from
// 6.2 to 5.2 TB/s on this B200 (tools/read_bw.cu "sweep": the slowdown is a
// step at the carve-out switch, not a function of the smem size).
constexpr size_t kFastCarveBytes = 196 * 1024;
// two-pass scan segments per CTA: 1 measured best at config 4 (each segment
// boundary costs a pipeline drain + flush; 2/4/8 per CTA: +1/+4/+11%)
constexpr uint64_t kSegsPerCta = 1;
#define K3_SEL_SCRATCH_BYTES ((size_t)kThreads * 11 * 4)  // select_rows_t8 masks
// 32-byte units per thread per load batch (x2 double-buffered): keeps
// ~128 KB of loads in flight per SM at 512 (4 x 128) or 768 threads/SM
// 32-byte units per thread per load group (two groups in flight). 256-bit
// codes (W = 8, the two-pass config-4 scan) stream best with three:
// config-4 retrieval 418 -> 398 us; 128-bit codes with two (three: config-3
// 57.6 -> 60.7 us, config-2 decode 49.8 -> 51.4 us; four: worse on all).
constexpr int kU = kThreads == 128 ? 4 : 2;
template <int W>
constexpr int units_for() { return W == 8 ? 3 : kU; }

__device__ __forceinline__ uint64_t gtimer() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// ------------------------------------------------------------ block scans
__device__ __forceinline__ uint64_t warp_incl_scan_u64(uint64_t v) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        uint64_t n = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += n;
    }
    return v;
}

// Exclusive scan over a 256-thread block; `total` receives the block sum.
__device__ __forceinline__ uint64_t block_excl_scan_u64(uint64_t v, uint64_t* s_warp,
                                                        uint64_t& total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint64_t incl = warp_incl_scan_u64(v);
    if (lane == 31) s_warp[warp] = incl;
    __syncthreads();
    if (warp == 0) {
        uint64_t x = lane < (kThreads / 32) ? s_warp[lane] : 0;
        uint64_t xi = warp_incl_scan_u64(x);
        if (lane < (kThreads / 32)) s_warp[lane] = xi - x;
        if (lane == (kThreads / 32) - 1) s_warp[kThreads / 32] = xi;
    }
    __syncthreads();
    const uint64_t r = incl - v + s_warp[warp];
    total = s_warp[kThreads / 32];
    __syncthreads();
    return r;
}

// In-place suffix sum over a[0..n) in shared memory: a[t] = sum_{b >= t} a[b].
__device__ void block_suffix_sum(uint32_t* a, uint32_t n, uint64_t* s_warp) {
    uint64_t carry = 0;
    for (uint32_t base = 0; base < n; base += kThreads) {
        const uint32_t i = base + threadIdx.x;  // i-th from the top
        const uint32_t t = n - 1 - i;
        const uint64_t v = i < n ? a[t] : 0;
        uint64_t tot;
        const uint64_t ex = block_excl_scan_u64(v, s_warp, tot);
        if (i < n) a[t] = (uint32_t)(carry + ex + v);
        carry += tot;
        __syncthreads();
    }
}

// Threshold of one problem from its (global) histogram: s_cum <- suffix
// sums, returns T (SPL_PLAN_SKIP when kk == 0, or when fewer than kk rows
// score >= from) and the tie quota. Bins below `from` are read as 0.
__device__ void problem_threshold(const uint32_t* tot, uint32_t L, uint32_t kk, uint32_t* s_cum,
                                  uint64_t* s_warp, uint32_t* s_T, uint32_t& T, uint32_t& quota,
                                  uint32_t from = 0) {
    for (uint32_t t = threadIdx.x; t <= L + 1; t += kThreads)
        s_cum[t] = (t <= L && t >= from) ? __ldcg(tot + t) : 0u;
    __syncthreads();
    block_suffix_sum(s_cum, L + 1, s_warp);
    if (threadIdx.x == 0) *s_T = SPL_PLAN_SKIP;
    __syncthreads();
    if (kk > 0)
        for (uint32_t t = threadIdx.x; t <= L; t += kThreads)
            if (s_cum[t] >= kk && s_cum[t + 1] < kk) *s_T = t;
    __syncthreads();
    T = *s_T;
    quota = (T == SPL_PLAN_SKIP) ? 0u : kk - s_cum[T + 1];
    __syncthreads();
}

// plan.w = 1: the stored u8 scores cannot decide this threshold (clamped
// L = 256 scores and T >= 255), k3_select recomputes them from the codes.
__device__ __forceinline__ uint32_t exact_flag(const K3Params& prm, uint32_t T) {
    return (prm.clamp8 && T != SPL_PLAN_SKIP && T >= 255u) ? 1u : 0u;
}

// Two-pass: plan every segment of problem p given (T, quota).
__device__ void plan_segments(const K3Params& prm, uint32_t p, uint32_t T, uint32_t quota,
                              uint64_t* s_warp) {
    const uint32_t L2 = prm.L + 2;
    const uint32_t c0 = seg_first(prm.g, p), c1 = seg_last(prm.g, p);
    uint64_t carry_gt = 0, carry_eq = 0;
    for (uint32_t base = c0; base <= c1; base += kThreads) {
        const uint32_t c = base + threadIdx.x;
        uint32_t gt = 0, eq = 0;
        if (c <= c1 && T != SPL_PLAN_SKIP) {
            const uint32_t* rec = prm.records + (uint64_t)(c + p) * L2;
            const uint32_t geT = __ldcg(rec + T), geT1 = __ldcg(rec + T + 1);
            gt = geT1;
            eq = geT - geT1;
        }
        uint64_t tot;
        const uint64_t ex = block_excl_scan_u64(((uint64_t)eq << 32) | gt, s_warp, tot);
        if (c <= c1) {
            const uint64_t gt_before = carry_gt + (ex & 0xffffffffu);
            const uint64_t eq_before = carry_eq + (ex >> 32);
            const uint64_t left = quota > eq_before ? quota - eq_before : 0;
            const uint32_t take = (uint32_t)(eq < left ? eq : left);
            const uint32_t off = (uint32_t)(gt_before + (eq_before < quota ? eq_before : quota));
            prm.plans[c + p] = make_uint4(T, off, take, exact_flag(prm, T));
        }
        carry_gt += tot & 0xffffffffu;
        carry_eq += tot >> 32;
    }
}

// Two-pass low-threshold fallback: plan the segments of problem p by
// counting score > T / == T over each segment's stored scores (T < 255).
template <typename ScoreT>
__device__ void plan_segments_recount(const K3Params& prm, uint32_t p, uint32_t nv, uint32_t T,
                                      uint32_t quota, uint64_t* s_warp) {
    const K3Geom& g = prm.g;
    const ScoreT* srow = reinterpret_cast<const ScoreT*>(prm.scores) + (uint64_t)p * g.n_pad;
    const uint64_t pbase = (uint64_t)p * g.pstride;
    uint64_t carry_gt = 0, carry_eq = 0;
    for (uint32_t c = seg_first(g, p); c <= seg_last(g, p); ++c) {
        const uint64_t lo_r = max((uint64_t)c * g.S, pbase) - pbase;
        const uint64_t hi_r = min(min(((uint64_t)c + 1) * g.S, pbase + g.pstride) - pbase, (uint64_t)nv);
        uint32_t gt = 0, eq = 0;
        if (T != SPL_PLAN_SKIP)
            for (uint64_t r = lo_r + threadIdx.x; r < hi_r; r += kThreads) {
                const uint32_t v = srow[r];
                gt += v > T;
                eq += v == T;
            }
        uint64_t tot;
        block_excl_scan_u64(((uint64_t)eq << 32) | gt, s_warp, tot);
        if (threadIdx.x == 0) {
            const uint64_t eeq = tot >> 32;
            const uint64_t left = quota > carry_eq ? quota - carry_eq : 0;
            const uint32_t take = (uint32_t)(eeq < left ? eeq : left);
            const uint32_t off = (uint32_t)(carry_gt + (carry_eq < quota ? carry_eq : quota));
            prm.plans[c + p] = make_uint4(T, off, take, 0u);
        }
        carry_gt += tot & 0xffffffffu;
        carry_eq += tot >> 32;
    }
}

// ------------------------------------------------------------ streaming
struct Unit32 {
    uint32_t w[8];
    __device__ __forceinline__ void load(const uint32_t* base, uint64_t unit) {
        const uint32_t* p = base + unit * 8;
        asm volatile(
            "ld.global.nc.L1::no_allocate.L2::evict_first.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
            : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3]), "=r"(w[4]), "=r"(w[5]),
              "=r"(w[6]), "=r"(w[7])
            : "l"(p));
    }
};

template <typename ScoreT, int R>
__device__ __forceinline__ void store_scores(ScoreT* dst, const uint32_t* s) {
    if constexpr (sizeof(ScoreT) * R == 1) {
        *reinterpret_cast<uint8_t*>(dst) = (uint8_t)s[0];
    } else if constexpr (sizeof(ScoreT) * R == 2) {
        uint32_t v = 0;
#pragma unroll
        for (int r = 0; r < R; ++r) v |= s[r] << (r * 8 * sizeof(ScoreT));
        *reinterpret_cast<uint16_t*>(dst) = (uint16_t)v;
    } else if constexpr (sizeof(ScoreT) * R == 4) {
        uint32_t v = 0;
#pragma unroll
        for (int r = 0; r < R; ++r) v |= s[r] << (r * 8 * sizeof(ScoreT));
        *reinterpret_cast<uint32_t*>(dst) = v;
    } else {
        uint64_t v = 0;
#pragma unroll
        for (int r = 0; r < R; ++r) v |= (uint64_t)s[r] << (r * 8 * sizeof(ScoreT));
        *reinterpret_cast<uint64_t*>(dst) = v;
    }
}

// Byte slot of thread t inside a 256-byte bin row of the private counters:
// the 32 lanes of a warp land in 32 distinct banks (lane*4), the 4 bytes of
// a bank word belong to 4 different warps. (Slot = t would put lanes
// 4i..4i+3 on one bank with different bins: a 4-way conflict per update.)
// The flush sums whole bin rows, so it does not depend on the mapping.
__device__ __forceinline__ uint32_t priv_slot(uint32_t t) {
    static_assert(kThreads % 128 == 0, "priv_slot maps 4 warps per 128-byte group");
    return (t & 31u) * 4u + ((t >> 5) & 3u) + (t >> 7) * 128u;
}
template <bool PRIV>
__device__ __forceinline__ void count_score(uint8_t* priv, uint32_t* hist32, uint32_t s) {
    if (PRIV)
        priv[s * kThreads + priv_slot(threadIdx.x)] += 1;
    else
        atomicAdd(hist32 + s, 1u);
}

// Add the private u8 counters [bins][kThreads] into hist32 and clear them.
static_assert(kThreads == 128 || kThreads == 256, "flush_priv row width");
__device__ void flush_priv(uint8_t* priv, uint32_t* hist32, uint32_t bins) {
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (uint32_t b = warp; b < bins; b += kThreads / 32) {
        uint32_t sum = 0;
        if constexpr (kThreads == 128) {  // 128 B = 32 x 4 B
            uint32_t* row = reinterpret_cast<uint32_t*>(priv + (size_t)b * kThreads);
            sum = __vsadu4(row[lane], 0u);
            row[lane] = 0u;
        } else {  // 256 B = 32 x 8 B
            uint2* row = reinterpret_cast<uint2*>(priv + (size_t)b * kThreads);
            const uint2 x = row[lane];
            sum = __vsadu4(x.x, 0u) + __vsadu4(x.y, 0u);
            row[lane] = make_uint2(0u, 0u);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
        if (lane == 0) hist32[b] += sum;
    }
    __syncthreads();
}

// Transposed on-chip layout of u8 scores (fused path): inside each 16-row
// vector, word i byte b holds row 4b + i, so OR-ing the per-word SWAR flag
// masks shifted by (7 - i) yields one flag bit per row in row order
// (select_rows_t8). Byte position of row j (relative to the 16-aligned a0):
__device__ __forceinline__ uint32_t tpos(uint32_t j) {
    return (j & ~15u) | ((j & 3u) << 2) | ((j >> 2) & 3u);
}

// One row's agreement score from W words (edge rows: plain loads).
template <int W>
__device__ __forceinline__ uint32_t row_score(const uint32_t* row, const uint32_t* q, uint32_t L) {
    uint32_t mism = 0;
#pragma unroll
    for (int w = 0; w < W; ++w) mism += __popc(__ldg(row + w) ^ q[w]);
    return L - mism;
}

// Stream rows [r0, r1) of one problem: scores into dst[row - dst_row0],
// counts into priv / hist32. Uniform control flow across the block (flushes
// sync the block). The body of the loop is check-free: rows before the first
// / after the last whole 32-byte unit are handled up front, and only the last
// iteration (pair) tests unit bounds. Offsets inside a piece are 32-bit.
template <int W, typename ScoreT, bool PRIV, bool DST_SMEM>
__device__ void stream_piece(const uint32_t* base, const uint32_t* qp, uint32_t L, uint64_t r0,
                             uint64_t r1, ScoreT* dst, uint64_t dst_row0, uint8_t* priv,
                             uint32_t* hist32, uint32_t bins, uint32_t lo) {
    // counters (priv rows / hist32 entries) are indexed by score - lo; scores
    // below lo are stored but not counted (lo = 0: full histogram)
    constexpr bool TR = DST_SMEM && sizeof(ScoreT) == 1;  // transposed layout (tpos)
    const int tid = threadIdx.x;
    if constexpr (W > 0) {
        constexpr int KU = units_for<W>();
        constexpr int R = 8 / W;  // rows per 32-byte unit
        constexpr bool kClamp = sizeof(ScoreT) == 1 && W == 8;
        uint32_t q[W];
#pragma unroll
        for (int w = 0; w < W; ++w) q[w] = __ldg(qp + w);
        // whole units [uh, ut); partial-unit rows [r0, uh*R) and [ut*R, r1)
        const uint64_t uh = (r0 + R - 1) / R, ut = r1 / R;
        {
            const uint64_t head_end = min(r1, uh * R);
            const uint64_t tail_beg = max(head_end, ut * R);
            const uint32_t nhead = (uint32_t)(head_end - r0), ntail = (uint32_t)(r1 - tail_beg);
            if ((uint32_t)tid < nhead + ntail) {
                const uint64_t row = (uint32_t)tid < nhead ? r0 + tid : tail_beg + (tid - nhead);
                const uint32_t sc = row_score<W>(base + row * W, q, L);
                const uint32_t sv = kClamp ? min(sc, 255u) : sc;
                if constexpr (TR)
                    dst[tpos((uint32_t)(row - dst_row0))] = (ScoreT)sv;
                else
                    dst[row - dst_row0] = (ScoreT)sv;
                if (sc >= lo) count_score<PRIV>(priv, hist32, sc - lo);
            }
        }
        if (ut <= uh) {
            if (PRIV) flush_priv(priv, hist32, bins);
            __syncthreads();
            return;
        }
        const uint32_t nu = (uint32_t)(ut - uh);
        const uint32_t* ubase = base + uh * 8 + (size_t)tid * 8;  // this thread's unit 0
        ScoreT* udst = dst + (uh * R - dst_row0) + (size_t)tid * R;  // its scores
        // private counters through 32-bit shared-window addresses hoisted out
        // of the loop (ld/st.shared.u8; asm volatile keeps their order)
        const uint32_t priv_s = (uint32_t)__cvta_generic_to_shared(priv) + priv_slot(tid);
        const uint32_t dst_s = DST_SMEM ? (uint32_t)__cvta_generic_to_shared(udst) : 0u;
        // transposed layout: row index of this thread's unit 0 relative to a0
        const uint32_t jb = (uint32_t)(uh * R - dst_row0) + (uint32_t)tid * R;
        const uint32_t dst0_s = TR ? (uint32_t)__cvta_generic_to_shared(dst) : 0u;
        constexpr uint32_t per_it = (uint32_t)kThreads * KU;
        const uint32_t nit = (nu + per_it - 1) / per_it;
        // private u8 counters: flush before any thread can add 256 to a bin
        // (each iteration adds at most KU * R per thread; iterations go in pairs)
        constexpr uint32_t kFlushPairs = (255 / (KU * R)) / 2 > 0 ? (255 / (KU * R)) / 2 : 1;
        Unit32 a[KU], b[KU];
        auto load = [&](Unit32* buf, uint32_t it, bool check) {
            const uint32_t* p = ubase + (size_t)it * per_it * 8;
#pragma unroll
            for (int j = 0; j < KU; ++j)
                if (!check || it * per_it + j * kThreads + tid < nu) buf[j].load(p, (uint32_t)j * kThreads);
        };
        auto count = [&](uint32_t sc) {
            if (sc < lo) return;
            if (PRIV) {
                const uint32_t addr = priv_s + (sc - lo) * kThreads;
                uint32_t v;
                asm volatile("ld.shared.u8 %0, [%1];" : "=r"(v) : "r"(addr));
                asm volatile("st.shared.u8 [%0], %1;" ::"r"(addr), "r"(v + 1));
            } else {
                atomicAdd(hist32 + (sc - lo), 1u);
            }
        };
        auto process_unit = [&](const Unit32& u, uint32_t it, int j) {
            uint32_t sc[R];
#pragma unroll
            for (int r = 0; r < R; ++r) {
                uint32_t mism = 0;
#pragma unroll
                for (int w = 0; w < W; ++w) mism += __popc(u.w[r * W + w] ^ q[w]);
                sc[r] = L - mism;
            }
            // u8 scores at L = 256: stored as min(score, 255) (exact for
            // every threshold <= 254; the counters below see the true score)
            uint32_t st[R];
#pragma unroll
            for (int r = 0; r < R; ++r) st[r] = kClamp ? min(sc[r], 255u) : sc[r];
            const size_t off = ((size_t)it * per_it + (size_t)j * kThreads) * R;
            if constexpr (TR) {
                // R consecutive rows from a multiple of R (R | 16): row r of
                // the unit sits 4 * (r % 4) + r / 4 bytes after tpos(first)
                const uint32_t ad = dst0_s + tpos(jb + (uint32_t)off);
#pragma unroll
                for (int r = 0; r < R; ++r)
                    asm volatile("st.shared.u8 [%0], %1;" ::"r"(ad + 4 * (r & 3) + (r >> 2)), "r"(st[r]));
            } else if constexpr (DST_SMEM) {
                uint32_t v = 0;
#pragma unroll
                for (int r = 0; r < R; ++r) v |= st[r] << (r * 8 * sizeof(ScoreT));
                const uint32_t ad = dst_s + (uint32_t)(off * sizeof(ScoreT));
                if constexpr (sizeof(ScoreT) * R == 1)
                    asm volatile("st.shared.u8 [%0], %1;" ::"r"(ad), "r"(v));
                else if constexpr (sizeof(ScoreT) * R == 2)
                    asm volatile("st.shared.u16 [%0], %1;" ::"r"(ad), "h"((unsigned short)v));
                else if constexpr (sizeof(ScoreT) * R == 4)
                    asm volatile("st.shared.u32 [%0], %1;" ::"r"(ad), "r"(v));
                else
                    store_scores<ScoreT, R>(udst + off, st);
            } else {
                store_scores<ScoreT, R>(udst + off, st);
            }
#pragma unroll
            for (int r = 0; r < R; ++r) count(sc[r]);
        };
        auto process_full = [&](const Unit32* buf, uint32_t it) {
#pragma unroll
            for (int j = 0; j < KU; ++j) process_unit(buf[j], it, j);
        };
        auto process_tail = [&](const Unit32* buf, uint32_t it) {
#pragma unroll
            for (int j = 0; j < KU; ++j)
                if (it * per_it + j * kThreads + tid < nu) process_unit(buf[j], it, j);
        };
        const uint32_t nfull = nu / per_it;  // iterations with every unit in range
        load(a, 0, nfull == 0);
        for (uint32_t it = 0; it < nit; it += 2) {
            if (it + 1 < nit) load(b, it + 1, it + 1 >= nfull);
            if (it < nfull) process_full(a, it); else process_tail(a, it);
            if (it + 1 < nit) {
                if (it + 2 < nit) load(a, it + 2, it + 2 >= nfull);
                if (it + 1 < nfull) process_full(b, it + 1); else process_tail(b, it + 1);
            }
            if (PRIV && ((it / 2 + 1) % kFlushPairs) == 0) flush_priv(priv, hist32, bins);
        }
    } else {
        // any W: 32-bit loads, one row per thread per step
        const uint32_t Wr = L / 32;
        uint32_t steps = 0;
        for (uint64_t r = r0 + tid; r - tid < r1; r += kThreads) {
            if (r < r1) {
                const uint32_t* row = base + r * Wr;
                uint32_t mism = 0;
                for (uint32_t w = 0; w < Wr; ++w) mism += __popc(__ldg(row + w) ^ __ldg(qp + w));
                const uint32_t s = L - mism;
                dst[r - dst_row0] = (ScoreT)(sizeof(ScoreT) == 1 ? min(s, 255u) : s);
                if (s >= lo) count_score<PRIV>(priv, hist32, s - lo);
            }
            if (PRIV && ++steps == 255) {
                flush_priv(priv, hist32, bins);
                steps = 0;
            }
        }
    }
    if (PRIV) flush_priv(priv, hist32, bins);
    __syncthreads();
}

// ------------------------------------------------------------ ordered select
// Per-row flags of 4 packed u8 / 2 packed u16 scores against a threshold.
// u8 (any byte value, incl. the clamped L = 256 scores): carry-free SWAR.
// With xl = w & 0x7f.., xh = w & 0x80..: for s <= 127, byte >= s iff bit 7 of
// (xl + 128 - s) | xh; for s >= 128, iff bit 7 of (xl + 256 - s) & xh (xl <=
// 127 keeps every byte sum below 256). The __vcmp*4 intrinsics are emulated
// on sm_100 and made the select issue-bound.
struct U8Cmp {
    uint32_t add, hi_or, hi_and;  // per-byte addend; xh OR-mask (s <= 127) / AND-mask (s >= 128)
    uint32_t never;               // s > 255: no byte qualifies
};
__device__ __forceinline__ U8Cmp u8cmp_ge(uint32_t s) {
    U8Cmp c;
    c.never = s > 255 ? 1u : 0u;
    if (s <= 127) {
        c.add = (128u - s) * 0x01010101u;
        c.hi_or = 0xFFFFFFFFu;
        c.hi_and = 0xFFFFFFFFu;
    } else {
        c.add = (256u - (s > 255 ? 255u : s)) * 0x01010101u;
        c.hi_or = 0u;
        c.hi_and = 0u;
    }
    return c;
}
// bit 7 of each byte = (byte >= s)
__device__ __forceinline__ uint32_t u8_ge(uint32_t xl, uint32_t xh, const U8Cmp& c) {
    const uint32_t t = xl + c.add;
    // s <= 127: t | xh ; s >= 128: t & xh
    const uint32_t r = c.hi_or ? (t | xh) : (t & xh);
    return c.never ? 0u : (r & 0x80808080u);
}
template <typename ScoreT>
struct WordCmp {
    U8Cmp ge, gt;   // u8
    uint32_t Tw;    // u16
};
template <typename ScoreT>
__device__ __forceinline__ WordCmp<ScoreT> make_wordcmp(uint32_t T) {
    WordCmp<ScoreT> c;
    c.ge = u8cmp_ge(T);
    c.gt = u8cmp_ge(T + 1);
    c.Tw = T * 0x00010001u;
    return c;
}
template <typename ScoreT>
__device__ __forceinline__ void word_flags(uint32_t w, const WordCmp<ScoreT>& c, uint32_t& gt,
                                           uint32_t& eq) {
    if constexpr (sizeof(ScoreT) == 1) {
        const uint32_t xl = w & 0x7F7F7F7Fu, xh = w & 0x80808080u;
        const uint32_t ge = u8_ge(xl, xh, c.ge), g = u8_ge(xl, xh, c.gt);
        // 0x80 flags of bytes 0..3 -> bits 0..3
        gt = ((g >> 7) * 0x01020408u) >> 24;
        eq = (((ge & ~g) >> 7) * 0x01020408u) >> 24;
    } else {
        const uint32_t g = __vcmpgtu2(w, c.Tw), e = __vcmpeq2(w, c.Tw);
        gt = (g & 1u) | ((g >> 15) & 2u);
        eq = (e & 1u) | ((e >> 15) & 2u);
    }
}

// Ordered compaction of rows [r0, r1) whose scores sit at sc[row - a0]
// (a0 = r0 rounded down to 16 rows; sc 16-byte aligned): keep score > T and
// the first `take` score == T rows, writing ascending row ids to out[0..).
// Each thread owns NG consecutive groups of 64 rows per round, all loads of
// a round issued before any is used (GLOBAL: the two-pass k3_select reads
// L2/DRAM, so a round is one memory latency; NG = 4 cuts the rounds of a
// 150 K-row segment from 10 to 3).
template <typename ScoreT, bool GLOBAL>
__device__ void select_rows(const ScoreT* sc, uint64_t a0, uint64_t r0, uint64_t r1, uint32_t T,
                            uint32_t take, uint32_t* out, uint64_t* s_warp) {
    constexpr int PER = 16 / sizeof(ScoreT);  // scores per 16-byte vector
    constexpr int NVG = 64 / PER;             // vectors per 64-row group
    constexpr int NG = 1;  // groups per thread per round (4: k3_select 43 -> 48 us at config 4)
    constexpr int CH = 64 * NG;               // rows per thread per round
    constexpr int SPW = 4 / sizeof(ScoreT);   // scores per word
    const WordCmp<ScoreT> Tw = make_wordcmp<ScoreT>(T);
    const int tid = threadIdx.x;
    const uint64_t round_rows = (uint64_t)kThreads * CH;
    uint64_t carry_gt = 0, carry_eq = 0;
    for (uint64_t base = a0; base < r1; base += round_rows) {
        const uint64_t my = base + (uint64_t)tid * CH;
        uint4 x[NG * NVG];
#pragma unroll
        for (int v = 0; v < NG * NVG; ++v) {
            const uint64_t at = my + (uint64_t)v * PER;
            x[v] = make_uint4(0, 0, 0, 0);
            if (at < r1) {
                const uint4* ptr = reinterpret_cast<const uint4*>(sc + (at - a0));
                x[v] = GLOBAL ? __ldcg(ptr) : *ptr;
            }
        }
        uint64_t gtm[NG], eqm[NG];
        uint32_t gt = 0, eq = 0;
#pragma unroll
        for (int gi = 0; gi < NG; ++gi) {
            gtm[gi] = 0;
            eqm[gi] = 0;
#pragma unroll
            for (int v = 0; v < NVG; ++v) {
                const uint4 xv = x[gi * NVG + v];
                const uint32_t ws[4] = {xv.x, xv.y, xv.z, xv.w};
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    uint32_t g, e;
                    word_flags<ScoreT>(ws[i], Tw, g, e);
                    gtm[gi] |= (uint64_t)g << (v * PER + i * SPW);
                    eqm[gi] |= (uint64_t)e << (v * PER + i * SPW);
                }
            }
            // rows outside [r0, r1)
            const uint64_t g0 = my + 64 * gi;
            const uint64_t lo = r0 > g0 ? r0 - g0 : 0;
            const uint64_t hi = r1 > g0 ? (r1 - g0 < 64 ? r1 - g0 : 64) : 0;
            uint64_t valid = hi >= 64 ? ~0ull : ((1ull << hi) - 1);
            valid &= lo >= 64 ? 0ull : ~((1ull << lo) - 1);
            gtm[gi] &= valid;
            eqm[gi] &= valid;
            gt += __popcll(gtm[gi]);
            eq += __popcll(eqm[gi]);
        }
        uint64_t tot;
        const uint64_t ex = block_excl_scan_u64(((uint64_t)eq << 32) | gt, s_warp, tot);
        if (gt | eq) {
            uint64_t eq_before = carry_eq + (ex >> 32);
            uint64_t pos = carry_gt + (ex & 0xffffffffu) + (eq_before < take ? eq_before : take);
#pragma unroll
            for (int gi = 0; gi < NG; ++gi) {
                uint64_t m = gtm[gi] | eqm[gi];
                const uint32_t rowb = (uint32_t)(my + 64 * gi);
                while (m) {
                    const int i = __ffsll((long long)m) - 1;
                    m &= m - 1;
                    if ((gtm[gi] >> i) & 1u) {
                        out[pos++] = rowb + i;
                    } else {
                        if (eq_before < take) out[pos++] = rowb + i;
                        ++eq_before;
                    }
                }
            }
        }
        carry_gt += tot & 0xffffffffu;
        carry_eq += tot >> 32;
    }
}

// Fused-path select over u8 scores in the transposed layout (tpos), L <= 128
// so every score is <= 128: with c = (128 - t) * 0x01010101, byte x >= t
// iff bit 7 of byte (x + c) is set, and x + c never carries into the next
// byte. Flags per word: (w + c) >> (7 - i) masked with 0x01010101 << i and
// OR-ed (IADD, SHF, LOP3), so bit 8b + i of a vector's mask is row 4b + i
// (row order = bit order). Same contract as select_rows.
// Each thread owns NV consecutive 16-row vectors per round; NV odd makes the
// per-lane stride (16 * NV bytes) hit 8 distinct 16-byte bank groups across
// any 8 lanes, so every LDS.128 is conflict-free (4 wavefronts). NV = 11
// covers the headline segment (40448 rows) in one round (one block scan);
// NV = 3 short segments (<= 12 K rows, the config-2 decode shape).
// The select is issue-bound (all CTAs of an SM select at once), so the
// per-vector work is kept to ~30 instructions: the stream zeroes the rows of
// the first / last vector outside [r0, r1), and a zero byte never reaches a
// threshold T >= 1, so only EDGE (T == 0: every row qualifies) masks them;
// the tie quota is resolved per thread (keep all / none), and only the one
// thread whose ties straddle `take` trims a vector; ids are emitted straight
// from the per-vector masks in registers.
// Output: when the CTA's `count` ids fit the shared-memory stage (stage_cap
// entries), they are compacted there and written to out[0..count) with
// coalesced stores at the end (the scattered 4-byte stores of the emission
// loop cost more than the compaction itself); the decode step's attention
// then reads them from the stage. Otherwise they go straight to out.
// PF (decode step): prefetch each emitted row's K and V lines into L2 (when
// pfk is set).
__device__ __forceinline__ uint32_t keep_lowest_bits(uint32_t e, uint32_t n) {
    uint32_t r = 0;
    for (uint32_t c = 0; c < n; ++c) {
        r |= e & (0u - e);
        e &= e - 1;
    }
    return r;
}

// Per-vector flags: gt = rows with score > T, ge = rows with score >= T (one
// bit per row, bit 8b + i <-> row 4b + i). EDGE (T == 0): every row inside
// [lo, hi) is >= T and nothing outside.
template <bool EDGE>
__device__ __forceinline__ void t8_flags(const uint8_t* sc, uint32_t at, uint32_t lo, uint32_t hi,
                                         uint32_t c_gt, uint32_t c_ge, uint32_t m_gt, uint32_t& g,
                                         uint32_t& ge) {
    uint4 x = make_uint4(0, 0, 0, 0);
    if (at < hi) x = *reinterpret_cast<const uint4*>(sc + at);
    const uint32_t w[4] = {x.x, x.y, x.z, x.w};
    g = 0;
    ge = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        g |= ((w[i] + c_gt) >> (7 - i)) & (0x01010101u << i);
        if constexpr (!EDGE) ge |= ((w[i] + c_ge) >> (7 - i)) & (0x01010101u << i);
    }
    g &= m_gt;
    if constexpr (EDGE) {
        uint32_t valid = 0;
        if (at < hi) {
            valid = 0x0F0F0F0Fu;
            if (at < lo || at + 16 > hi)
                for (uint32_t j = 0; j < 16; ++j)
                    if (at + j < lo || at + j >= hi) valid &= ~(1u << (8 * (j >> 2) + (j & 3)));
        }
        ge = valid;
        g &= valid;
    }
}

// Rolled loops (the select runs once per CTA per launch, so its instructions
// come cold from L2: ncu showed it stalled on instruction fetch, not on
// arithmetic), two passes over the scores (count, then emit), both ~40
// instructions of loop body.
template <int NV, bool PF = false, bool EDGE = false>
__device__ void select_rows_t8(const uint8_t* sc, uint64_t a0, uint64_t r0, uint64_t r1,
                               uint32_t T, uint32_t take, uint32_t* out, uint64_t* s_warp,
                               uint64_t* tr, const char* pfk, const char* pfv, uint32_t pfb,
                               uint32_t* stage, uint32_t stage_cap, uint32_t count,
                               uint32_t* masks) {
    constexpr int CH = 16 * NV;  // rows per thread per round
    const bool staged = stage != nullptr && count <= stage_cap;  // uniform
    // T >= 128: no row is > T (c_gt masked off); EDGE is the T == 0 case
    const uint32_t c_ge = EDGE ? 0u : (128u - T) * 0x01010101u;
    const uint32_t c_gt = T < 128 ? (127u - T) * 0x01010101u : 0u;
    const uint32_t m_gt = T < 128 ? 0x0F0F0F0Fu : 0u;
    const uint32_t lo = (uint32_t)(r0 - a0), hi = (uint32_t)(r1 - a0);  // rows [lo, hi)
    const uint32_t rb = (uint32_t)a0;  // output row ids are a0 + offset (32-bit)
    const int tid = threadIdx.x;
    const uint32_t round_rows = (uint32_t)kThreads * CH;
    uint32_t carry_gt = 0, carry_eq = 0;
    for (uint32_t base = 0; base < hi; base += round_rows) {
        const uint32_t my = base + (uint32_t)tid * CH;
        uint32_t gt = 0, eq = 0, nzv = 0;  // nzv: vectors holding candidate rows
#pragma unroll
        for (int v = 0; v < NV; ++v) {
            uint32_t g, ge;
            t8_flags<EDGE>(sc, my + 16u * v, lo, hi, c_gt, c_ge, m_gt, g, ge);
            gt += __popc(g);
            eq += __popc(ge & ~g);
            nzv |= (ge != 0u ? 1u : 0u) << v;
            // both masks use bits 8b + i (i < 4): pack > T in the low, == T in the high nibbles
            if (ge) masks[(uint32_t)tid * NV + v] = g | ((ge & ~g) << 4);
        }
        if (tr && threadIdx.x == 0) { tr[9] = gtimer(); tr[13] = clock64(); }
        uint64_t tot;
        const uint64_t ex = block_excl_scan_u64(((uint64_t)eq << 32) | gt, s_warp, tot);
        if (tr && threadIdx.x == 0) { tr[10] = gtimer(); tr[14] = clock64(); }
        if (gt | eq) {
            const uint32_t eb = carry_eq + (uint32_t)(ex >> 32);  // ties before this thread's rows
            uint32_t pos = carry_gt + (uint32_t)ex + (eb < take ? eb : take);
            // ties this thread keeps: all (~0), none (0), or the first `left`
            uint32_t left = eb >= take ? 0u : (eb + eq <= take ? 0xFFFFFFFFu : take - eb);
            const uint32_t rowb = rb + my;
            while (nzv) {  // only the vectors with candidates, in row order
                const int v = __ffs(nzv) - 1;
                nzv &= nzv - 1;
                const uint32_t pk = masks[(uint32_t)tid * NV + v];
                const uint32_t g = pk & 0x0F0F0F0Fu;
                uint32_t e = left == 0u ? 0u : (pk >> 4) & 0x0F0F0F0Fu;
                if (left - 1u < 0xFFFFFFFEu) {  // the straddling thread
                    const uint32_t ne = __popc(e);
                    if (left < ne) e = keep_lowest_bits(e, left);
                    left -= left < ne ? left : ne;
                }
                uint32_t m = g | e;
                while (m) {
                    const uint32_t bb = __ffs(m) - 1;
                    m &= m - 1;
                    const uint32_t id = rowb + 16u * v + 4 * (bb >> 3) + (bb & 7);
                    if (staged)
                        stage[pos] = id;
                    else
                        out[pos] = id;
                    ++pos;
                    if constexpr (PF) {  // warm L2 for the attention gather (decode step)
                        if (!pfk) continue;
                        const char* kr = pfk + (uint64_t)id * pfb;
                        const char* vr = pfv + (uint64_t)id * pfb;
                        for (uint32_t b = 0; b < pfb; b += 128) {
                            asm volatile("prefetch.global.L2 [%0];" ::"l"(kr + b));
                            asm volatile("prefetch.global.L2 [%0];" ::"l"(vr + b));
                        }
                    }
                }
            }
        }
        carry_gt += (uint32_t)tot;
        carry_eq += (uint32_t)(tot >> 32);
    }
    if (staged) {
        __syncthreads();
        for (uint32_t i = tid; i < count; i += kThreads) out[i] = stage[i];
    }
    if (tr && threadIdx.x == 0) { tr[11] = gtimer(); tr[15] = clock64(); }
}

// ------------------------------------------------------------------ scan
__device__ __forceinline__ uint32_t ld_acquire(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
// Spin (one thread) until *p >= need. A wait that outlives 2 s means some
// CTA of the problem was never scheduled: flag SPL_DEV_ERR_STALL and give up
// rather than hang the stream (results of that launch are then invalid).
__device__ void wait_count(const uint32_t* p, uint32_t need, uint32_t* dev_err) {
    if (ld_acquire(p) >= need) return;
    const uint64_t t0 = gtimer();
    while (ld_acquire(p) < need) {
        __nanosleep(64);
        if (gtimer() - t0 > 2000000000ull) {
            raise_dev_err(dev_err, SPL_DEV_ERR_STALL);
            return;
        }
    }
}

// Ordered compaction with scores recomputed from the codes (plan.w = 1: the
// stored u8 scores are clamped and T >= 255). Same contract as select_rows.
__device__ void select_rows_exact(const K3Params& prm, uint32_t p, uint64_t r0, uint64_t r1,
                                  uint32_t T, uint32_t take, uint32_t* out, uint64_t* s_warp) {
    const uint32_t W = prm.W;
    const uint32_t* q = prm.qcodes + (uint64_t)p * W;
    const uint32_t* base = prm.codes + (uint64_t)p * prm.stride_rows * W;
    uint64_t carry_gt = 0, carry_eq = 0;
    for (uint64_t b = r0; b < r1; b += kThreads) {
        const uint64_t r = b + threadIdx.x;
        uint32_t gt = 0, eq = 0;
        if (r < r1) {
            uint32_t mism = 0;
            for (uint32_t w = 0; w < W; ++w) mism += __popc(__ldg(base + r * W + w) ^ __ldg(q + w));
            const uint32_t sc = prm.L - mism;
            gt = sc > T;
            eq = sc == T;
        }
        uint64_t tot;
        const uint64_t ex = block_excl_scan_u64(((uint64_t)eq << 32) | gt, s_warp, tot);
        const uint64_t eq_before = carry_eq + (ex >> 32);
        const uint64_t pos = carry_gt + (ex & 0xffffffffu) + (eq_before < take ? eq_before : take);
        if (gt || (eq && eq_before < take)) out[pos] = (uint32_t)r;
        carry_gt += tot & 0xffffffffu;
        carry_eq += tot >> 32;
    }
}

// Two-pass scan: CTAs walk the segments grid-stride (segment = S rows of the
// virtual row space; several per CTA, so all CTAs sweep the problems in order
// and problems complete progressively); per segment: stream, private counts
// -> record + problem histogram; the CTA completing a problem plans it.
template <int W, typename ScoreT, bool PRIV>
__global__ void __launch_bounds__(kThreads, 3) k3_scan(K3Params prm) {
    extern __shared__ __align__(16) uint8_t smem[];
    __shared__ uint64_t s_warp[kThreads / 32 + 1];
    __shared__ uint32_t s_flag, s_T;
    const uint32_t L = prm.L;
    const uint32_t bins = L + 1;
    const uint32_t hlo = prm.hist_lo;  // counted window [hlo, L] (0: every bin)
    const uint32_t wbins = bins - hlo;
    const uint32_t Wr = (W > 0) ? (uint32_t)W : prm.W;
    const size_t priv_bytes = PRIV ? (((size_t)wbins * kThreads + 15) & ~size_t(15)) : 0;
    uint8_t* priv = smem;
    uint32_t* hist32 = reinterpret_cast<uint32_t*>(smem + priv_bytes);  // [bins + 1]
    const int tid = threadIdx.x;
    const K3Geom& g = prm.g;

    // zero the counters once (flush_priv re-zeroes them)
    pdl_trigger();
    if constexpr (PRIV)
        for (uint32_t i = tid; i < priv_bytes / 16; i += kThreads)
            reinterpret_cast<uint4*>(priv)[i] = make_uint4(0, 0, 0, 0);
    pdl_wait();

    for (uint32_t seg = blockIdx.x; seg < g.G; seg += gridDim.x) {
    const uint64_t g0 = (uint64_t)seg * g.S;
    const uint64_t g1 = min(g0 + g.S, g.total);
    const uint32_t p_first = (uint32_t)(g0 / g.pstride);
    for (uint32_t p = p_first; p < g.P && (uint64_t)p * g.pstride < g1; ++p) {
        const uint64_t pbase = (uint64_t)p * g.pstride;
        const uint64_t lo = max(g0, pbase) - pbase;
        const uint64_t hi = min(g1, pbase + g.pstride) - pbase;
        uint32_t nv = prm.n_valid[p / prm.nvalid_div];
        if (nv > g.n_max) {
            if (tid == 0) raise_dev_err(prm.dev_err, SPL_DEV_ERR_DIMENSION);
            nv = (uint32_t)g.n_max;
        }
        const uint64_t r0 = lo, r1 = min(hi, (uint64_t)nv);
        for (uint32_t i = tid; i <= bins; i += kThreads) hist32[i] = 0;
        __syncthreads();

        if (r0 < r1) {
            const uint32_t* qp = prm.qcodes + (uint64_t)p * Wr;
            const uint32_t* base = prm.codes + (uint64_t)p * prm.stride_rows * Wr;
            ScoreT* dst = reinterpret_cast<ScoreT*>(prm.scores) + (uint64_t)p * g.n_pad;
            stream_piece<W, ScoreT, PRIV, false>(base, qp, L, r0, r1, dst, 0, priv, hist32 + hlo,
                                                 wbins, hlo);
        }
        __syncthreads();
        // raw counts -> global per-problem histogram (integer atomics: the
        // sums are order-independent, so results stay deterministic)
        uint32_t* tot = prm.tot_hist + (uint64_t)p * prm.tot_stride;
        for (uint32_t b = hlo + tid; b < bins; b += kThreads)
            if (hist32[b]) atomicAdd(tot + b, hist32[b]);
        __syncthreads();
        block_suffix_sum(hist32, bins, s_warp);  // hist32[bins] stays 0
        uint32_t* rec = prm.records + (uint64_t)(seg + p) * (L + 2);
        for (uint32_t t = tid; t < L + 2; t += kThreads) rec[t] = hist32[t];

        if (!prm.shard) {
            __threadfence();
            __syncthreads();
            if (tid == 0) {
                const uint32_t nseg = seg_last(g, p) - seg_first(g, p) + 1;
                const uint32_t prev = atomicAdd(prm.counters + p, 1u);
                s_flag = (prev + 1 == nseg) ? 1u : 0u;
            }
            __syncthreads();
            if (s_flag) {
                __threadfence();
                const uint32_t kk = prm.k < nv ? prm.k : nv;
                uint32_t T, quota;
                problem_threshold(tot, L, kk, hist32, s_warp, &s_T, T, quota, hlo);
                const bool low = kk > 0 && T == SPL_PLAN_SKIP && hlo > 0;
                if (low) {
                    // Fewer than kk rows scored >= lo: count the bins below
                    // the window from the stored scores (exact below 255),
                    // take T again and plan the segments by recounting.
                    // Exact for any data; slow only for such problems.
                    const ScoreT* srow = reinterpret_cast<const ScoreT*>(prm.scores) + (uint64_t)p * g.n_pad;
                    for (uint32_t t = tid; t < hlo; t += kThreads) hist32[t] = 0u;
                    __syncthreads();
                    for (uint32_t r = tid; r < nv; r += kThreads) {
                        const uint32_t v = srow[r];
                        if (v < hlo) atomicAdd(hist32 + v, 1u);
                    }
                    __syncthreads();
                    for (uint32_t t = tid; t < hlo; t += kThreads) tot[t] = hist32[t];
                    __threadfence();
                    __syncthreads();
                    problem_threshold(tot, L, kk, hist32, s_warp, &s_T, T, quota);
                }
                for (uint32_t t = tid; t <= L; t += kThreads) tot[t] = 0u;  // self-reset
                if (low)
                    plan_segments_recount<ScoreT>(prm, p, nv, T, quota, s_warp);
                else
                    plan_segments(prm, p, T, quota, s_warp);
                if (tid == 0) {
                    prm.cnt_out[p] = kk;
                    prm.counters[p] = 0u;
                }
            }
        }
        __syncthreads();
    }
    }
}

// ------------------------------------------------------------ peer exchange
// Exchange area of one rank: u64 entries {value, epoch} (NCCL "LL"-style:
// the epoch tag travels in the same aligned 8-byte store as the value, so a
// reader that sees the current epoch sees the value, and no system-scope
// fence is needed on either side — a MEMBAR.SYS under the streaming load cost
// ~13 us). S = L + 2 entries per (rank, problem): bins 0..L and, at L + 1,
// the sender's valid row count. Double-buffered by epoch parity (a rank can
// run at most one call ahead of a peer: it cannot finish call i + 1 before
// that peer pushed its call-(i + 1) histograms, which it does only after
// finishing call i):  recv [2][R][Pmax][S] x u64.
__host__ __device__ __forceinline__ uint64_t xslot(uint32_t R, uint32_t Pmax, uint32_t S,
                                                   uint32_t par, uint32_t r, uint32_t p) {
    return (((uint64_t)par * R + r) * Pmax + p) * S;
}
__host__ __device__ __forceinline__ uint64_t xwords(uint32_t R, uint32_t Pmax, uint32_t S) {
    return 2ull * 2ull * R * Pmax * S;  // u32 words
}
__device__ __forceinline__ void st_tagged(uint32_t* p, uint32_t v, uint32_t tag) {
    asm volatile("st.volatile.global.v2.u32 [%0], {%1, %2};" ::"l"(p), "r"(v), "r"(tag) : "memory");
}
__device__ __forceinline__ uint2 ld_tagged(const uint32_t* p) {
    uint2 r;
    asm volatile("ld.volatile.global.v2.u32 {%0, %1}, [%2];" : "=r"(r.x), "=r"(r.y) : "l"(p) : "memory");
    return r;
}
// One thread: spin until entry p carries `tag`; returns its value. 2 s watchdog.
__device__ uint32_t wait_tagged(const uint32_t* p, uint32_t tag, uint32_t* dev_err) {
    uint2 e = ld_tagged(p);
    if (e.y == tag) return e.x;
    const uint64_t t0 = gtimer();
    while ((e = ld_tagged(p)).y != tag) {
        __nanosleep(32);
        if (gtimer() - t0 > 2000000000ull) {
            raise_dev_err(dev_err, SPL_DEV_ERR_STALL);
            return 0;
        }
    }
    return e.x;
}
// Block: push bins [b0, b1) of this rank's problem histogram (tot, complete
// at GPU scope) into slot (rank, p) of every rank's exchange area.
__device__ void shard_push(const K3Params& prm, uint32_t epoch, const uint32_t* tot, uint32_t p,
                           uint32_t b0, uint32_t b1, bool with_count, uint32_t nv_local) {
    const uint32_t S = prm.L + 2, par = epoch & 1u;
    __threadfence();
    for (uint32_t r = 0; r < prm.R; ++r) {
        uint32_t* dst = prm.peer_bufs[r] + 2 * xslot(prm.R, prm.Pmax, S, par, prm.rank, p);
        for (uint32_t t = b0 + threadIdx.x; t < b1; t += kThreads)
            st_tagged(dst + 2 * t, __ldcg(tot + t), epoch);
        if (with_count && threadIdx.x == 0) st_tagged(dst + 2 * (prm.L + 1), nv_local, epoch);
    }
}
// Block: the global plan of problem p from all ranks' delivered histograms
// (bins >= from; the same integer arithmetic as spl_plan_shard). Collects
// the R x (bins [from, L] + count) entries into `mat` (shared, R x (L + 2)
// words; entries below `from` keep what an earlier round stored), waiting
// on each entry's epoch tag. Outputs are uniform across the block.
// T = SPL_PLAN_SKIP: kk == 0, or fewer than kk rows score >= from (the
// caller then runs the low-bin round).
struct ShardPlanOut {
    uint32_t T, take, count, off, kk;
};
__device__ ShardPlanOut shard_global_plan(const K3Params& prm, uint32_t epoch, uint32_t p,
                                          uint32_t from, uint32_t to, uint32_t* mat,
                                          uint32_t* s_cum, uint64_t* s_warp,
                                          unsigned long long* s_red, uint32_t* s_aux) {
    const uint32_t L = prm.L, S = L + 2, par = epoch & 1u;
    const uint32_t* base = prm.own_buf + 2 * xslot(prm.R, prm.Pmax, S, par, 0, p);
    const uint64_t rs = 2ull * prm.Pmax * S;  // rank stride (u32 words)
    // entries [from, to) of every rank (+ the count at L + 1 when to == L + 2)
    const uint32_t span = to - from;
    for (uint32_t i = threadIdx.x; i < prm.R * span; i += kThreads) {
        const uint32_t r = i / span, t = from + i % span;
        mat[r * S + t] = wait_tagged(base + r * rs + 2 * t, epoch, prm.dev_err);
    }
    if (threadIdx.x < 4) s_red[threadIdx.x] = 0;
    if (threadIdx.x == 0) s_aux[0] = SPL_PLAN_SKIP;
    __syncthreads();
    uint64_t nloc = 0;
    for (uint32_t r = threadIdx.x; r < prm.R; r += kThreads) nloc += mat[r * S + L + 1];
    if (nloc) atomicAdd(&s_red[0], (unsigned long long)nloc);
    const uint32_t lo = (to == L + 2) ? from : 0;  // bins counted so far: [lo, L]
    for (uint32_t t = threadIdx.x; t <= L + 1; t += kThreads) {
        uint32_t G = 0;
        if (t >= lo && t <= L)
            for (uint32_t r = 0; r < prm.R; ++r) G += mat[r * S + t];
        s_cum[t] = G;
    }
    __syncthreads();
    const uint64_t n = s_red[0];
    ShardPlanOut o{SPL_PLAN_SKIP, 0, 0, 0, (uint32_t)(prm.k < n ? prm.k : n)};
    if (o.kk == 0) return o;
    block_suffix_sum(s_cum, L + 1, s_warp);  // s_cum[t] = #(score >= t) over bins >= lo
    for (uint32_t t = threadIdx.x; t <= L; t += kThreads)
        if (s_cum[t] >= o.kk && s_cum[t + 1] < o.kk) s_aux[0] = t;
    __syncthreads();
    o.T = s_aux[0];
    if (o.T == SPL_PLAN_SKIP) return o;
    const uint64_t quota = o.kk - s_cum[o.T + 1];
    uint64_t gtb = 0, gtm = 0;
    for (uint32_t t = o.T + threadIdx.x; t <= L; t += kThreads) {
        uint32_t before = 0;
        for (uint32_t r = 0; r < prm.rank; ++r) before += mat[r * S + t];
        const uint32_t mine = mat[prm.rank * S + t];
        if (t > o.T) {
            gtb += before;
            gtm += mine;
        } else {
            s_aux[1] = before;
            s_aux[2] = mine;
        }
    }
    if (gtb) atomicAdd(&s_red[1], (unsigned long long)gtb);
    if (gtm) atomicAdd(&s_red[2], (unsigned long long)gtm);
    __syncthreads();
    const uint64_t eq_before = s_aux[1], eq_mine = s_aux[2];
    const uint64_t left = quota > eq_before ? quota - eq_before : 0;
    o.take = (uint32_t)(eq_mine < left ? eq_mine : left);
    o.count = (uint32_t)(s_red[2] + o.take);
    o.off = (uint32_t)(s_red[1] + (eq_before < quota ? eq_before : quota));
    __syncthreads();
    return o;
}

// ------------------------------------------------ partial exchange (sharded decode)
// Second area of every rank's peer buffer (after the histograms): per (epoch
// parity, source rank, problem) D + 2 tagged u64 entries {value bits, epoch}
// = (m, l, o[D]) of that rank's partial attention. Same LL protocol as the
// histograms: value and tag land in one 8-byte store, double-buffered by
// parity (a rank cannot run two calls ahead of a peer).
constexpr uint32_t kPartDMax = 256;  // head dims the exchange supports
__host__ __device__ __forceinline__ uint64_t part_slot(uint32_t R, uint32_t Pmax, uint32_t par,
                                                       uint32_t r, uint32_t p) {
    return 2ull * ((((uint64_t)par * R + r) * Pmax + p) * (kPartDMax + 2));  // u32 words
}
__host__ __device__ __forceinline__ uint64_t part_words(uint32_t R, uint32_t Pmax) {
    return part_slot(R, Pmax, 2, 0, 0);
}
// Entry i of this rank's partial of problem p -> every rank's area.
__device__ __forceinline__ void part_push(const K3Params& prm, uint32_t epoch, uint32_t p,
                                          uint32_t i, float v) {
    const uint64_t at = prm.part_off + part_slot(prm.R, prm.Pmax, epoch & 1u, prm.rank, p) + 2 * i;
    for (uint32_t r = 0; r < prm.R; ++r) st_tagged(prm.peer_bufs[r] + at, __float_as_uint(v), epoch);
}
// Entry i of rank r's partial of problem p, from this rank's own area.
__device__ __forceinline__ float part_wait(const K3Params& prm, uint32_t epoch, uint32_t r,
                                           uint32_t p, uint32_t i) {
    const uint64_t at = prm.part_off + part_slot(prm.R, prm.Pmax, epoch & 1u, r, p) + 2 * i;
    return __uint_as_float(wait_tagged(prm.own_buf + at, epoch, prm.dev_err));
}
// Thread `dim` (< D) of the CTA that finished problem p on this rank: push
// the rank's (M, L, o[dim]) (thread 0 also M and L), collect all R ranks'
// and return the normalised output (flash-decoding log-sum-exp combine).
__device__ float part_exchange_combine(const K3Params& prm, uint32_t epoch, uint32_t p,
                                       uint32_t dim, float M, float Ls, float o) {
    if (dim == 0) {
        part_push(prm, epoch, p, 0, M);
        part_push(prm, epoch, p, 1, Ls);
    }
    part_push(prm, epoch, p, 2 + dim, o);
    float Mx = -INFINITY;
    for (uint32_t r = 0; r < prm.R; ++r) Mx = fmaxf(Mx, part_wait(prm, epoch, r, p, 0));
    float acc = 0.0f, Lt = 0.0f;
    for (uint32_t r = 0; r < prm.R; ++r) {
        const float m = part_wait(prm, epoch, r, p, 0);
        if (m == -INFINITY) continue;
        const float f = exp2f(m - Mx);
        Lt = fmaf(part_wait(prm, epoch, r, p, 1), f, Lt);
        acc = fmaf(part_wait(prm, epoch, r, p, 2 + dim), f, acc);
    }
    return acc / Lt;
}

// Sharded decode step, unfused form (head dims other than 128): this rank's
// partial attention partials [P][D + 2] (spl_sparse_attend_partial) are
// exchanged with the peer group and combined; one CTA of D threads per
// problem. The epoch is the one the preceding k3_fused<SHARD> call stored.
__global__ void k5_peer_combine(K3Params prm, const float* partials, uint32_t D, float* out) {
    const uint32_t p = blockIdx.x, dim = threadIdx.x;
    const uint32_t epoch = __ldcg(prm.epoch_ptr);
    const float* pp = partials + (uint64_t)p * (D + 2);
    if (dim < D) out[(uint64_t)p * D + dim] = part_exchange_combine(prm, epoch, p, dim, pp[0], pp[1], pp[2 + dim]);
}

// ------------------------------------------------------------ fused attend
// Shared-memory layout of the private-counter region once the stream is over
// (decode step, k3_fused<.., ATT>): [attention merge / combine scratch:
// kAttScratch floats] [emitted ids]. The select compacts the CTA's ids there
// when they fit (att_ids_cap), so the attention that follows does not read
// them back from L2.
constexpr uint32_t kAttScratchWords = 2 * 8 + 8 * 128;  // warp merge (the combine needs less)
__device__ __forceinline__ uint32_t att_ids_off_words(uint32_t) { return kAttScratchWords; }
template <bool ATT>
__device__ __forceinline__ uint32_t* att_ids(uint8_t* priv, size_t priv_bytes, uint32_t nv_sel) {
    if constexpr (!ATT) return nullptr;
    return reinterpret_cast<uint32_t*>(priv) + att_ids_off_words(nv_sel);
}
template <bool ATT>
__device__ __forceinline__ uint32_t att_ids_cap(size_t priv_bytes, uint32_t nv_sel) {
    if constexpr (!ATT) return 0;
    // the select's packed masks (nv_sel x kThreads words) sit at the end
    const size_t words = priv_bytes / 4 - (size_t)nv_sel * kThreads, off = att_ids_off_words(nv_sel);
    return words > off ? (uint32_t)(words - off) : 0u;
}

// Decode step, after a CTA compacted its rows of problem p (count entries at
// idx_out[p][off..), the first ids_cap of them also in shared memory): attend
// them (sparse_attention, attention_eval.cpp:234-264) right here instead of
// in a K4 launch. The CTA whose segment holds the own row nv - 1 adds it when
// it was not selected (:249-260). The 8 warps split the CTA's entries
// (warp_attend: 8-row batches, the K and V slices of a batch in flight
// together), merge (m, l, o) in shared memory and write the segment's
// partial; the CTA completing the problem's last segment merges the nseg
// partials (log-sum-exp, every load of the merge issued in one round) into
// att_out[p]. Every CTA of the problem calls this (those with no rows write
// an empty partial). scratch: kAttScratchWords floats.
// SHARD (sequence-sharded decode step): the problem's combined partial is
// this rank's only; it is exchanged with the other ranks through peer memory
// (part_exchange_combine) and every rank writes the same final output.
template <typename KV, bool SHARD>
__device__ void fused_attend(const K3Params& prm, uint32_t p, uint32_t seg, uint32_t c0,
                             uint32_t nseg, uint32_t nv, bool owner, uint64_t off, uint32_t count,
                             float* scratch, const uint32_t* sids, uint32_t ids_cap,
                             uint32_t* s_flag, uint32_t epoch) {
    constexpr int E = 4, D = 128, NW = kThreads / 32;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    float qv[E];
#pragma unroll
    for (int e = 0; e < E; ++e) qv[e] = __ldg(prm.att_q + (uint64_t)p * D + lane * E + e) * prm.att_qscale;
    const uint32_t* gids = prm.idx_out + (uint64_t)p * prm.idx_stride + off;
    const bool smem_ids = count <= ids_cap;
    __syncthreads();  // the emitted ids (shared / global) and the select's masks are complete
    uint32_t extra = kAttInv;
    if (owner && nv > 0) {
        const uint32_t last = count == 0 ? kAttInv : (smem_ids ? sids[count - 1] : __ldcg(gids + count - 1));
        if (last != nv - 1) extra = nv - 1;
    }
    const uint32_t total = count + (extra != kAttInv ? 1u : 0u);
    const uint32_t per = (total + NW - 1) / NW;
    const uint32_t j0 = min(total, warp * per), j1 = min(total, j0 + per);
    const uint64_t rb = (uint64_t)p * prm.stride_rows;
    const KV* kbase = reinterpret_cast<const KV*>(prm.pf_k) + rb * D;
    const KV* vbase = reinterpret_cast<const KV*>(prm.pf_v) + rb * D;
    float m = -INFINITY, lsum = 0.0f, o[E];
#pragma unroll
    for (int e = 0; e < E; ++e) o[e] = 0.0f;
    if (j0 < j1) {
        if (smem_ids)
            warp_attend<E, KV, true>(kbase, vbase, sids, count, extra, j0, j1, qv, m, lsum, o);
        else
            warp_attend<E, KV, false>(kbase, vbase, gids, count, extra, j0, j1, qv, m, lsum, o);
    }
    const float l = attend_lsum_total(lsum);
    // merge the warps -> this segment's partial (m, l, o)
    float* s_m = scratch;            // [NW]
    float* s_l = scratch + NW;       // [NW]
    float* s_o = scratch + 2 * NW;   // [NW][D]
    __syncthreads();  // every warp is done with the ids (they may share the region)
    if (lane == 0) {
        s_m[warp] = m;
        s_l[warp] = l;
    }
#pragma unroll
    for (int e = 0; e < E; ++e) s_o[warp * D + lane * E + e] = o[e];
    __syncthreads();
    float M = -INFINITY;
#pragma unroll
    for (int w = 0; w < NW; ++w) M = fmaxf(M, s_m[w]);
    float* part = prm.att_part + (uint64_t)(seg + p) * (D + 2);
    if (tid < D) {
        float acc = 0.0f;
#pragma unroll
        for (int w = 0; w < NW; ++w)
            if (s_m[w] != -INFINITY) acc += s_o[w * D + tid] * exp2f(s_m[w] - M);
        part[2 + tid] = acc;
    } else if (tid == D) {
        float Ls = 0.0f;
#pragma unroll
        for (int w = 0; w < NW; ++w)
            if (s_m[w] != -INFINITY) Ls += s_l[w] * exp2f(s_m[w] - M);
        part[0] = M;
        part[1] = Ls;
    }
    __threadfence();
    __syncthreads();
    if (tid == 0) *s_flag = (atomicAdd(prm.att_cnt + p, 1u) + 1 == nseg) ? 1u : 0u;
    __syncthreads();
    if (!*s_flag) return;
    // last segment of p: combine the nseg partials (slots c + p, c in [c0, c0 + nseg)).
    // Thread (half, dim) takes the partials i = half, half + 2, ...; their m,
    // l and o[dim] are loaded together (one round), scaled after the max.
    __threadfence();
    const float* base = prm.att_part + (uint64_t)(c0 + p) * (D + 2);
    const uint32_t dim = tid & (D - 1), half = tid / D;
    constexpr int kMaxPer = 8;  // partials per thread per round
    float Mx = -INFINITY, Lx = 0.0f, acc = 0.0f;
    for (uint32_t i0 = half; i0 < nseg; i0 += 2 * kMaxPer) {
        float mv[kMaxPer], lv[kMaxPer], ov[kMaxPer];
#pragma unroll
        for (int j = 0; j < kMaxPer; ++j) {
            const uint32_t i = i0 + 2 * j;
            mv[j] = -INFINITY;
            lv[j] = ov[j] = 0.0f;
            if (i < nseg) {
                const float* pp = base + (uint64_t)i * (D + 2);
                mv[j] = __ldcg(pp);
                lv[j] = __ldcg(pp + 1);
                ov[j] = __ldcg(pp + 2 + dim);
            }
        }
        float Mn = Mx;
#pragma unroll
        for (int j = 0; j < kMaxPer; ++j) Mn = fmaxf(Mn, mv[j]);
        const float r = Mx == -INFINITY ? 0.0f : exp2f(Mx - Mn);
        acc *= r;
        Lx *= r;
#pragma unroll
        for (int j = 0; j < kMaxPer; ++j) {
            const float sc = mv[j] == -INFINITY ? 0.0f : exp2f(mv[j] - Mn);
            acc = fmaf(ov[j], sc, acc);
            Lx = fmaf(lv[j], sc, Lx);
        }
        Mx = Mn;
    }
    // merge the two halves
    float* s_hm = scratch;           // [2] per-half max (all threads of a half agree)
    float* s_hl = scratch + 2;       // [2]
    float* s_ha = scratch + 4;       // [2][D]
    __syncthreads();
    if (dim == 0) {
        s_hm[half] = Mx;
        s_hl[half] = Lx;
    }
    s_ha[half * D + dim] = acc;
    __syncthreads();
    if (tid < D) {
        const float M2 = fmaxf(s_hm[0], s_hm[1]);
        const float f0 = s_hm[0] == -INFINITY ? 0.0f : exp2f(s_hm[0] - M2);
        const float f1 = s_hm[1] == -INFINITY ? 0.0f : exp2f(s_hm[1] - M2);
        const float Lt = s_hl[0] * f0 + s_hl[1] * f1;
        const float ov = s_ha[tid] * f0 + s_ha[D + tid] * f1;
        if constexpr (SHARD)
            prm.att_out[(uint64_t)p * D + tid] = part_exchange_combine(prm, epoch, p, tid, M2, Lt, ov);
        else
            prm.att_out[(uint64_t)p * D + tid] = ov / Lt;
    }
    if (tid == 0) prm.att_cnt[p] = 0u;  // self-reset for the next launch / graph replay
}

// ------------------------------------------------------------ fused
// Single-launch path for caches whose scores fit on chip (the headline
// 32 x 512K case). Contiguous segments, a whole number per problem (G <= SMs
// x 3 CTAs at 80 registers), scores kept in shared memory:
// stream -> segment record + per-problem histogram of the window [L/2, L]
// (atomics) -> wait for the problem's other segments -> T / tie quota from
// the problem histogram (low-bin fallback when T < L/2), output offset from
// the earlier segments' records -> compact the rows from shared memory.
// Shared memory stays <= 196 KB/SM: above that the driver must choose the
// 228 KB carve-out and LDG streaming loses ~16% (tools/read_bw.cu).
#define K3_STAMP(i) \
    if (prm.trace && threadIdx.x == 0) prm.trace[blockIdx.x * 16 + (i)] = gtimer()

// SHARD: one rank of a sequence-sharded cache. The CTA completing a
// problem's local histogram pushes it to every rank's exchange area (peer
// memory over NVLink), every CTA of the problem waits for all ranks' pushes,
// takes the global threshold / tie quota / this rank's share and offset
// (shard_global_plan) and compacts its rows as usual — one launch, no
// host-side collective. Local positions, plus out_offset[p] into the global
// list (rank order = index order, as in spl_shard_select).
// ATT (decode step): also attend the selected rows (fused_attend; KV = K/V
// cache element type, head dim 128), writing the attention output.
template <int W, typename ScoreT, bool SHARD = false, bool PF = false, bool ATT = false,
          typename KV = __nv_bfloat16>
__global__ void __launch_bounds__(kThreads, 3) k3_fused(K3Params prm) {
    extern __shared__ __align__(16) uint8_t smem[];
    __shared__ uint64_t s_warp[kThreads / 32 + 1];
    __shared__ uint32_t s_flag, s_T;
    __shared__ unsigned long long s_red[4];
    __shared__ uint32_t s_aux[4];
    const uint32_t L = prm.L;
    const uint32_t bins = L + 1;
    const uint32_t lo = prm.hist_lo;        // counted window [lo, L]
    const uint32_t wbins = bins - lo;
    // the private counters double as select_rows_t8's scratch afterwards
    const size_t priv_counters = ((size_t)wbins * kThreads + 15) & ~size_t(15);
    const size_t priv_bytes =
        priv_counters > K3_SEL_SCRATCH_BYTES ? priv_counters : K3_SEL_SCRATCH_BYTES;
    const size_t hist_bytes = (((size_t)(bins + 1) * 4) + 15) & ~size_t(15);
    uint8_t* priv = smem;
    uint32_t* hist32 = reinterpret_cast<uint32_t*>(smem + priv_bytes);                // [bins + 1]
    uint32_t* s_cum = reinterpret_cast<uint32_t*>(smem + priv_bytes + hist_bytes);    // [bins + 1]
    uint8_t* sregion = smem + priv_bytes + 2 * hist_bytes;
    const int tid = threadIdx.x;
    const K3Geom& g = prm.g;
    K3_STAMP(0);
    if (prm.trace && tid == 0) {
        uint32_t smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        prm.trace[(uint64_t)blockIdx.x * 16 + 6] = smid;
    }
    // The readiness waits below need the CTAs of a problem to run together:
    // the plan keeps G <= usable SMs x CTAs/SM (occupancy API). Plain launch
    // by default: CTAs are dispatched in index order and a problem's segments
    // are neighbours, so a concurrent kernel holding SMs only delays the
    // retrieval (tests/test_gpu_coresidency.py). SM-limited contexts (green
    // contexts, MPS caps: detected at spl_ctx_create) or SPL_K3_COOP=1 launch
    // cooperatively (a cooperative launch costs ~3 us more per graph replay);
    // if the driver refuses, the two-pass kernels run instead. The watchdog in
    // wait_count turns any remaining hang into a device error. (Arrival
    // tickets would remove the dispatch-order assumption, but measured +4 us
    // on the back-to-back headline: segment-to-SM placement changes per launch.)
    const uint32_t seg = blockIdx.x;
    pdl_trigger();
    for (uint32_t i = tid; i < priv_bytes / 16; i += kThreads)
        reinterpret_cast<uint4*>(priv)[i] = make_uint4(0, 0, 0, 0);
    pdl_wait();  // query codes / appended code rows come from the previous kernel
    K3_STAMP(2);
    // SHARD: this call's epoch = the group's device-side counter + 1 (the
    // last CTA stores it back), so CUDA-graph replays advance it too
    uint32_t epoch = 0;
    if constexpr (SHARD) {
        epoch = __ldcg(prm.epoch_ptr) + 1u;
        // 0 marks never-written entries; wrap 0xFFFFFFFF -> 2 (not 1) so the
        // parity keeps alternating between consecutive calls
        if (epoch == 0) epoch = 2;
    }

    const uint64_t g0 = (uint64_t)seg * g.S;
    const uint64_t g1 = min(g0 + g.S, g.total);
    const uint32_t p_first = (uint32_t)(g0 / g.pstride);
    uint32_t region_off = 0;  // byte offset of the current piece's scores

    for (uint32_t p = p_first; p < g.P && (uint64_t)p * g.pstride < g1; ++p) {
        const uint64_t pbase = (uint64_t)p * g.pstride;
        const uint64_t lo_r = max(g0, pbase) - pbase;
        const uint64_t hi_r = min(g1, pbase + g.pstride) - pbase;
        uint32_t nv = prm.n_valid[p / prm.nvalid_div];
        if (nv > g.n_max) {
            if (tid == 0) raise_dev_err(prm.dev_err, SPL_DEV_ERR_DIMENSION);
            nv = (uint32_t)g.n_max;
        }
        const uint64_t r0 = lo_r, r1 = min(hi_r, (uint64_t)nv);
        for (uint32_t i = tid; i <= bins; i += kThreads) hist32[i] = 0;
        __syncthreads();
        if (r0 < r1) {
            const uint64_t a0 = r0 & ~uint64_t(15);
            ScoreT* dst = reinterpret_cast<ScoreT*>(sregion + region_off);
            region_off += (uint32_t)((((r1 - a0) * sizeof(ScoreT)) + 15) & ~uint64_t(15));
            stream_piece<W, ScoreT, true, true>(prm.codes + (uint64_t)p * prm.stride_rows * W,
                                                prm.qcodes + (uint64_t)p * W, L, r0, r1, dst, a0,
                                                priv, hist32 + lo, wbins, lo);
            if constexpr (sizeof(ScoreT) == 1) {
                // zero the unused rows of the first / last 16-row vector: the
                // SWAR compares of select_rows_t8 assume bytes <= 128, and
                // left-over shared memory could carry into a valid row's byte
                const uint32_t head = (uint32_t)(r0 - a0), end = (uint32_t)(r1 - a0);
                const uint32_t pad_end = (end + 15u) & ~15u;
                if ((uint32_t)tid < head) dst[tpos(tid)] = 0;
                if (end + tid < pad_end) dst[tpos(end + tid)] = 0;
            }
        }
        __syncthreads();
        uint32_t* tot = prm.tot_hist + (uint64_t)p * prm.tot_stride;
        for (uint32_t b = lo + tid; b < bins; b += kThreads)
            if (hist32[b]) atomicAdd(tot + b, hist32[b]);
        __syncthreads();
        // suffix-cumulative record; below the window it repeats rec[lo]
        block_suffix_sum(hist32, bins, s_warp);  // hist32[bins] stays 0
        uint32_t* rec = prm.records + (uint64_t)(seg + p) * (L + 2);
        for (uint32_t t = tid; t < L + 2; t += kThreads) rec[t] = hist32[t];
        // publish: this segment of problem p is complete (record + histogram)
        __threadfence();
        __syncthreads();
        if (tid == 0) {
            const uint32_t prev = atomicAdd(prm.counters + p, 1u);
            s_flag = prev + 1 == seg_last(g, p) - seg_first(g, p) + 1 ? 1u : 0u;
        }
        if constexpr (SHARD) {
            __syncthreads();
            if (s_flag) shard_push(prm, epoch, tot, p, lo, bins, true, nv);  // the local histogram is complete
        }
    }
    K3_STAMP(1);

    // ---------------- plan + select from shared memory
    region_off = 0;
    for (uint32_t p = p_first; p < g.P && (uint64_t)p * g.pstride < g1; ++p) {
        const uint64_t pbase = (uint64_t)p * g.pstride;
        const uint64_t lo_r = max(g0, pbase) - pbase;
        const uint64_t hi_r = min(g1, pbase + g.pstride) - pbase;
        uint32_t nv = prm.n_valid[p / prm.nvalid_div];
        if (nv > g.n_max) nv = (uint32_t)g.n_max;
        const uint64_t r0 = lo_r, r1 = min(hi_r, (uint64_t)nv);
        const uint32_t kk = prm.k < nv ? prm.k : nv;
        const uint32_t nseg = seg_last(g, p) - seg_first(g, p) + 1;
        const uint64_t a0 = r0 & ~uint64_t(15);
        const ScoreT* sc = reinterpret_cast<const ScoreT*>(sregion + region_off);
        if (r0 < r1) region_off += (uint32_t)((((r1 - a0) * sizeof(ScoreT)) + 15) & ~uint64_t(15));
        // wait only for the segments of THIS problem (all resident: see the
        // ticket note above), not for the whole grid
        if (tid == 0) wait_count(prm.counters + p, nseg, prm.dev_err);
        __syncthreads();
        uint32_t* tot = prm.tot_hist + (uint64_t)p * prm.tot_stride;
        const uint32_t c0 = seg_first(g, p);
        // window bins only: CTAs that take the fallback below add the low
        // bins to `tot` while others may still be reading it, and every CTA
        // of the problem must reach the same decision
        uint32_t T, quota;
        ShardPlanOut sp{};
        // SHARD: all ranks' histograms land in the private-counter region (free
        // now; the plan checked R x (L + 2) words fit)
        uint32_t* mat = reinterpret_cast<uint32_t*>(priv);
        if constexpr (SHARD) {
            sp = shard_global_plan(prm, epoch, p, lo, L + 2, mat, s_cum, s_warp, s_red, s_aux);
            T = sp.T;
            quota = sp.take;  // this rank's ties
        } else {
            problem_threshold(tot, L, kk, s_cum, s_warp, &s_T, T, quota, lo);
        }
        if ((SHARD ? sp.kk : kk) > 0 && T == SPL_PLAN_SKIP) {
            // Fewer than kk rows scored >= lo, so T < lo: every CTA of this
            // problem (the decision is the same for all of them) counts its
            // rows below the window from shared memory, completes its record
            // and the problem histogram, then T is taken again. Exact for any
            // data; only slower for problems whose k-th score is below L/2.
            for (uint32_t t = tid; t <= bins; t += kThreads) hist32[t] = 0;
            __syncthreads();
            if (r0 < r1)
                for (uint64_t r = r0 + tid; r < r1; r += kThreads) {
                    const uint32_t v = sizeof(ScoreT) == 1 ? sc[tpos((uint32_t)(r - a0))] : sc[r - a0];
                    if (v < lo) atomicAdd(hist32 + v, 1u);
                }
            __syncthreads();
            for (uint32_t b = tid; b < lo; b += kThreads)
                if (hist32[b]) atomicAdd(tot + b, hist32[b]);
            __syncthreads();
            block_suffix_sum(hist32, lo, s_warp);
            uint32_t* rec = prm.records + (uint64_t)(seg + p) * (L + 2);
            const uint32_t at_lo = __ldcg(rec + lo);
            for (uint32_t t = tid; t < lo; t += kThreads) rec[t] = at_lo + hist32[t];
            __threadfence();
            __syncthreads();
            if (tid == 0) {
                const uint32_t prev = atomicAdd(prm.counters2 + p, 1u);
                s_flag = prev + 1 == nseg ? 1u : 0u;
            }
            __syncthreads();
            if constexpr (SHARD) {
                if (s_flag) shard_push(prm, epoch, tot, p, 0, lo, false, 0);  // low bins of all local segments
            }
            if (tid == 0) wait_count(prm.counters2 + p, nseg, prm.dev_err);
            __syncthreads();
            if constexpr (SHARD) {
                sp = shard_global_plan(prm, epoch, p, 0, lo, mat, s_cum, s_warp, s_red, s_aux);
                T = sp.T;
                quota = sp.take;
            } else {
                problem_threshold(tot, L, kk, s_cum, s_warp, &s_T, T, quota);
            }
        }
        K3_STAMP(3);
        if (tid == 0 && seg == c0) {
            if constexpr (SHARD) {
                prm.cnt_out[p] = T == SPL_PLAN_SKIP ? 0u : sp.count;
                prm.out_offset[p] = sp.off;
            } else {
                prm.cnt_out[p] = kk;
            }
        }
        uint64_t off = 0;
        uint32_t my_count = 0;
        if (r0 < r1 && T != SPL_PLAN_SKIP) {
            // (gt, eq) of the earlier segments of this problem, from their records
            uint64_t gt_before = 0, eq_before = 0;
            for (uint32_t cb = c0; cb < seg; cb += kThreads) {
                const uint32_t c = cb + tid;
                uint32_t gtv = 0, eqv = 0;
                if (c < seg) {
                    const uint32_t* r = prm.records + (uint64_t)(c + p) * (L + 2);
                    const uint32_t geT = __ldcg(r + T), geT1 = __ldcg(r + T + 1);
                    gtv = geT1;
                    eqv = geT - geT1;
                }
                uint64_t totv;
                block_excl_scan_u64(((uint64_t)eqv << 32) | gtv, s_warp, totv);
                gt_before += totv & 0xffffffffu;
                eq_before += totv >> 32;
            }
            K3_STAMP(4);
            const uint32_t* own = prm.records + (uint64_t)(seg + p) * (L + 2);
            const uint64_t eq_mine = (uint64_t)__ldcg(own + T) - __ldcg(own + T + 1);
            const uint64_t left = quota > eq_before ? quota - eq_before : 0;
            const uint32_t take = (uint32_t)(eq_mine < left ? eq_mine : left);
            off = gt_before + (eq_before < quota ? eq_before : quota);
            my_count = __ldcg(own + T + 1) + take;
            K3_STAMP(8);
            if (prm.trace && threadIdx.x == 0) prm.trace[blockIdx.x * 16 + 12] = clock64();
            if constexpr (sizeof(ScoreT) == 1) {
                uint32_t* o = prm.idx_out + (uint64_t)p * prm.idx_stride + off;
                uint64_t* trp = prm.trace ? prm.trace + (uint64_t)blockIdx.x * 16 : nullptr;
                const uint64_t pf_off = (uint64_t)p * prm.stride_rows * prm.pf_row_bytes;
                const bool pf_emit = prm.pf_k && !ATT;  // the decode step attends the rows itself
                const char* pfk = pf_emit ? prm.pf_k + pf_off : nullptr;
                const char* pfv = pf_emit ? prm.pf_v + pf_off : nullptr;
                const uint8_t* sc8 = reinterpret_cast<const uint8_t*>(sc);
                const uint32_t pfb = prm.pf_row_bytes;
                const bool nv3 = r1 - a0 <= (uint64_t)kThreads * 16 * 3;  // uniform
                // stage for the emitted ids: the decode step's id region (its
                // attention reads them there), else the whole free counter region
                uint32_t* stg = ATT ? att_ids<ATT>(priv, priv_bytes, nv3 ? 3 : 11) : nullptr;
                // per-thread packed candidate masks (kThreads x NV words) behind
                // the stage in the free counter region
                const uint32_t nvw = (nv3 ? 3u : 11u) * kThreads;
                uint32_t* msk = reinterpret_cast<uint32_t*>(priv) + (priv_bytes / 4 - nvw);
                const uint32_t cap = ATT ? att_ids_cap<ATT>(priv_bytes, nv3 ? 3 : 11)
                                         : (uint32_t)(priv_bytes / 4 - nvw);
                if (nv3) {
                    if (T == 0)
                        select_rows_t8<3, PF, true>(sc8, a0, r0, r1, T, take, o, s_warp, trp, pfk, pfv, pfb, stg, cap, my_count, msk);
                    else
                        select_rows_t8<3, PF, false>(sc8, a0, r0, r1, T, take, o, s_warp, trp, pfk, pfv, pfb, stg, cap, my_count, msk);
                } else {
                    if (T == 0)
                        select_rows_t8<11, PF, true>(sc8, a0, r0, r1, T, take, o, s_warp, trp, pfk, pfv, pfb, stg, cap, my_count, msk);
                    else
                        select_rows_t8<11, PF, false>(sc8, a0, r0, r1, T, take, o, s_warp, trp, pfk, pfv, pfb, stg, cap, my_count, msk);
                }
            }
            else
                select_rows<ScoreT, false>(sc, a0, r0, r1, T, take,
                                           prm.idx_out + (uint64_t)p * prm.idx_stride + off, s_warp);
        }
        if constexpr (ATT) {
            K3_STAMP(7);
            const bool owner = prm.att_own && r0 < r1 && r1 == (uint64_t)nv;  // holds row nv - 1
            const uint32_t nvs = (r1 - a0 <= (uint64_t)kThreads * 16 * 3) ? 3u : 11u;  // select's NV
            fused_attend<KV, SHARD>(prm, p, seg, c0, nseg, nv, owner, off, my_count,
                                    reinterpret_cast<float*>(priv), att_ids<ATT>(priv, priv_bytes, nvs),
                                    att_ids_cap<ATT>(priv_bytes, nvs), &s_flag, epoch);
        }
    }
    K3_STAMP(5);

    // ---------------- completion: the last CTA resets the shared state
    __threadfence();
    __syncthreads();
    if (tid == 0) s_flag = (atomicAdd(prm.sync + 1, 1u) + 1 == gridDim.x) ? 1u : 0u;
    __syncthreads();
    if (s_flag) {
        __threadfence();
        for (uint64_t i = tid; i < (uint64_t)g.P * prm.tot_stride; i += kThreads) prm.tot_hist[i] = 0u;
        for (uint32_t i = tid; i < g.P; i += kThreads) {
            prm.counters[i] = 0u;
            prm.counters2[i] = 0u;
        }
        if (tid == 0) {
            prm.sync[0] = 0u;
            prm.sync[1] = 0u;
            if constexpr (SHARD) *prm.epoch_ptr = epoch;
        }
    }
}

// ---------------------------------------------------------------- select
template <typename ScoreT>
__global__ void __launch_bounds__(kThreads, 3) k3_select(K3Params prm, uint32_t* idx,
                                                      uint64_t idx_stride) {
    __shared__ uint64_t s_warp[kThreads / 32 + 1];
    const K3Geom& g = prm.g;
    pdl_trigger();
    pdl_wait();
    const uint64_t g0 = (uint64_t)blockIdx.x * g.S;
    const uint64_t g1 = min(g0 + g.S, g.total);
    for (uint32_t p = (uint32_t)(g0 / g.pstride); p < g.P && (uint64_t)p * g.pstride < g1; ++p) {
        const uint64_t pbase = (uint64_t)p * g.pstride;
        const uint64_t lo = max(g0, pbase) - pbase;
        const uint64_t hi = min(g1, pbase + g.pstride) - pbase;
        uint32_t nv = prm.n_valid[p / prm.nvalid_div];
        if (nv > g.n_max) nv = (uint32_t)g.n_max;
        const uint64_t r0 = lo, r1 = min(hi, (uint64_t)nv);
        const uint4 plan = prm.plans[blockIdx.x + p];
        if (plan.x == SPL_PLAN_SKIP || r0 >= r1) continue;  // uniform across the block
        if (plan.w) {
            select_rows_exact(prm, p, r0, r1, plan.x, plan.z, idx + (uint64_t)p * idx_stride + plan.y,
                              s_warp);
            continue;
        }
        const ScoreT* srow = reinterpret_cast<const ScoreT*>(prm.scores) + (uint64_t)p * g.n_pad;
        const uint64_t a0 = r0 & ~uint64_t(15);
        select_rows<ScoreT, true>(srow + a0, a0, r0, r1, plan.x, plan.z,
                                  idx + (uint64_t)p * idx_stride + plan.y, s_warp);
    }
}

// Shard planning: one CTA per problem, from all ranks' histograms. The same
// integer arithmetic as spl_plan_shard (spl_plan.cuh, the host form the CPU
// tests check), spread over the block: thread t owns score bin t (summing it
// over ranks), a block suffix sum finds T, and block reductions give this
// rank's tie share and output offset. (Run by one thread it walked
// R x (L + 1) global counters serially: 52 us at R = 8.)
__global__ void __launch_bounds__(kThreads) k3_shard_plan(K3Params prm, const uint32_t* all_hist,
                                                          uint32_t R, uint32_t rank,
                                                          uint32_t* out_offset) {
    __shared__ uint64_t s_warp[kThreads / 32 + 1];
    extern __shared__ uint32_t s_G[];            // [L + 2] global count per bin, then suffix sums
    __shared__ unsigned long long s_red[4];       // n, gt_before, gt_mine, (unused)
    __shared__ uint32_t s_T, s_eqb, s_eqm;
    const uint32_t p = blockIdx.x;
    const uint32_t L = prm.L;
    const uint64_t rstride = (uint64_t)prm.g.P * (L + 1);
    const uint32_t* h = all_hist + (uint64_t)p * (L + 1);
    if (threadIdx.x < 4) s_red[threadIdx.x] = 0;
    if (threadIdx.x == 0) s_T = SPL_PLAN_SKIP;
    for (uint32_t t = threadIdx.x; t <= L + 1; t += kThreads) s_G[t] = 0;
    __syncthreads();
    uint64_t n_loc = 0;
    for (uint32_t t = threadIdx.x; t <= L; t += kThreads) {
        uint32_t G = 0;
        for (uint32_t r = 0; r < R; ++r) G += __ldg(h + r * rstride + t);
        s_G[t] = G;
        n_loc += G;
    }
    if (n_loc) atomicAdd(&s_red[0], (unsigned long long)n_loc);
    __syncthreads();
    const uint64_t n = s_red[0];
    const uint32_t kk = (uint32_t)(prm.k < n ? prm.k : n);
    if (kk > 0) {
        block_suffix_sum(s_G, L + 1, s_warp);  // s_G[t] = #(score >= t), s_G[L+1] = 0
        for (uint32_t t = threadIdx.x; t <= L; t += kThreads)
            if (s_G[t] >= kk && s_G[t + 1] < kk) s_T = t;
        __syncthreads();
    }
    const uint32_t T = s_T;
    uint32_t take = 0, count = 0, off = 0;
    if (T != SPL_PLAN_SKIP) {
        const uint64_t quota = kk - s_G[T + 1];
        uint64_t gtb = 0, gtm = 0;
        for (uint32_t t = threadIdx.x; t <= L; t += kThreads) {
            uint32_t before = 0;
            for (uint32_t r = 0; r < rank; ++r) before += __ldg(h + r * rstride + t);
            const uint32_t mine = __ldg(h + (uint64_t)rank * rstride + t);
            if (t > T) {
                gtb += before;
                gtm += mine;
            } else if (t == T) {
                s_eqb = before;
                s_eqm = mine;
            }
        }
        if (gtb) atomicAdd(&s_red[1], (unsigned long long)gtb);
        if (gtm) atomicAdd(&s_red[2], (unsigned long long)gtm);
        __syncthreads();
        const uint64_t eq_before = s_eqb, eq_mine = s_eqm;
        const uint64_t left = quota > eq_before ? quota - eq_before : 0;
        take = (uint32_t)(eq_mine < left ? eq_mine : left);
        count = (uint32_t)(s_red[2] + take);
        off = (uint32_t)(s_red[1] + (eq_before < quota ? eq_before : quota));
    }
    plan_segments(prm, p, T, take, s_warp);
    if (threadIdx.x == 0) {
        prm.cnt_out[p] = T == SPL_PLAN_SKIP ? 0u : count;
        if (out_offset) out_offset[p] = off;
    }
}

// ------------------------------------------------------------ host side
spl_status ensure_buffer(spl_ctx* ctx, void** buf, size_t* have, size_t bytes, bool zero,
                         cudaStream_t s, const char* what) {
    if (*have >= bytes && *buf) return SPL_OK;
    if (stream_capturing(s))
        return fail(ctx, SPL_E_STATE,
                    std::string(what) + ": workspace too small during stream capture; call "
                                        "spl_reserve before capturing");
    if (*buf) {
        cudaStreamSynchronize(s);
        cudaFree(*buf);
        *buf = nullptr;
        *have = 0;
    }
    size_t want = std::max(bytes, (size_t)256);
    SPL_CUDA_TRY(ctx, cudaMalloc(buf, want));
    if (zero) {
        // zeroed on the caller's stream and completed before any kernel of
        // any stream can see the buffer (a legacy-stream cudaMemset is not
        // ordered before work on non-blocking streams)
        SPL_CUDA_TRY(ctx, cudaMemsetAsync(*buf, 0, want, s));
        SPL_CUDA_TRY(ctx, cudaStreamSynchronize(s));
    }
    *have = want;
    return SPL_OK;
}

namespace {

size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

// two-pass plan (also the sharded flow)
struct K3Plan {
    K3Geom g;
    bool vec;
    bool priv;
    size_t smem;
    size_t score_bytes;
    uint32_t hist_lo;  // counted score window [hist_lo, L]
    bool clamp8;       // two-pass u8 scores at L = 256 hold min(score, 255)
    uint32_t grid;     // two-pass scan CTAs (<= g.G segments, grid-stride)
};

template <int W, typename ScoreT, bool PRIV>
const void* scan_fn() {
    return reinterpret_cast<const void*>(&k3_scan<W, ScoreT, PRIV>);
}
template <typename ScoreT, bool PRIV>
const void* pick_w(uint32_t W) {
    switch (W) {
        case 1: return scan_fn<1, ScoreT, PRIV>();
        case 2: return scan_fn<2, ScoreT, PRIV>();
        case 4: return scan_fn<4, ScoreT, PRIV>();
        case 8: return scan_fn<8, ScoreT, PRIV>();
        default: return scan_fn<0, ScoreT, PRIV>();  // any W, 32-bit loads
    }
}
const void* pick_scan(const K3Plan& pl, uint32_t L) {
    const uint32_t W = pl.vec ? L / 32 : 0;
    if (pl.score_bytes == 1) return pl.priv ? pick_w<uint8_t, true>(W) : pick_w<uint8_t, false>(W);
    return pl.priv ? pick_w<uint16_t, true>(W) : pick_w<uint16_t, false>(W);
}

bool vec_ok(const void* codes, uint64_t stride_rows, uint32_t W) {
    return W <= 8 && 8 % W == 0 && (reinterpret_cast<uintptr_t>(codes) % 32) == 0 &&
           (stride_rows * W * 4) % 32 == 0;
}

// Two-pass geometry. `single` (one-GPU retrieval, planned in-kernel):
//  - private counters over the window [L/2, L] only when the full range
//    would not fit 3 CTAs/SM under the fast carve-out (the planner counts
//    the low bins from the stored scores if T < L/2, see k3_scan);
//  - u8 scores up to L = 256, clamped to 255 at L = 256 (half the score
//    traffic of u16; thresholds >= 255 re-read the codes, see exact_flag).
// The sharded flow keeps full histograms (they are all-gathered) and u16
// scores above L = 255.
spl_status make_plan(spl_ctx* ctx, uint32_t P, uint64_t n_max, uint32_t L, const void* codes,
                     uint64_t stride_rows, K3Plan* out, bool single = false) {
    K3Plan pl{};
    const uint32_t W = L / 32;
    pl.vec = vec_ok(codes, stride_rows, W);
    pl.score_bytes = (L <= 255 || (single && L == 256)) ? 1 : 2;
    pl.clamp8 = single && L == 256;
    const size_t hist_b = align_up((size_t)(L + 2) * 4, 16);
    if (single && (align_up((size_t)(L + 1) * kThreads, 16) + hist_b + 1024) * 3 > kFastCarveBytes)
        pl.hist_lo = L / 2;
    pl.priv = (size_t)(L + 1 - pl.hist_lo) * kThreads <= 96 * 1024;
    const uint64_t total = (uint64_t)P * n_max;
    pl.smem = (pl.priv ? align_up((size_t)(L + 1 - pl.hist_lo) * kThreads, 16) : 0) + hist_b;
    const void* fn = pick_scan(pl, L);
    SPL_CUDA_TRY(ctx, cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)pl.smem));
    // keep the SM's shared memory under the fast carve-out: streaming reads
    // lose ~16% with the 228 KB one (tools/read_bw.cu "sweep")
    SPL_CUDA_TRY(ctx, cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout,
                                           (int)(kFastCarveBytes * 100 / (228 * 1024))));
    int per_sm = 0;
    SPL_CUDA_TRY(ctx, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kThreads, pl.smem));
    if (per_sm < 1) per_sm = 1;
    const uint64_t G_target = (uint64_t)ctx->num_sms * per_sm;
    // kSegsPerCta segments per CTA, walked grid-stride (SPL_K3_SEGS overrides
    // it for experiments)
    uint64_t spc = kSegsPerCta;
    if (const char* e = getenv("SPL_K3_SEGS")) spc = std::max(1, atoi(e));  // experiments
    uint64_t S = (total + G_target * spc - 1) / (G_target * spc);
    S = align_up(std::max<uint64_t>(S, 1024), 256);
    pl.g.n_max = n_max;
    pl.g.pstride = n_max;
    pl.g.total = total;
    pl.g.S = S;
    pl.g.G = (uint32_t)((total + S - 1) / S);
    pl.grid = (uint32_t)std::min<uint64_t>(pl.g.G, G_target);
    pl.g.P = P;
    pl.g.n_pad = align_up(n_max, 64);
    *out = pl;
    return SPL_OK;
}

// fused plan: geometry + launch shape when the scores fit on chip
struct K3FPlan {
    K3Plan pl;
    size_t smem;
    const void* fn;
};

template <int W, typename ScoreT, bool SHARD = false, bool PF = false, bool ATT = false,
          typename KV = __nv_bfloat16>
const void* fused_fn() {
    return reinterpret_cast<const void*>(&k3_fused<W, ScoreT, SHARD, PF, ATT, KV>);
}

// att: 0 = plain retrieval, 1 / 2 = decode step attending bf16 / f32 K/V rows
// (k3_fused<4, u8, false, true, true, KV>; L = 128 only)
spl_status make_fused_plan(spl_ctx* ctx, uint32_t P, uint64_t n_max, uint32_t L, const void* codes,
                           uint64_t stride_rows, bool* ok, K3FPlan* out, bool shard = false,
                           bool pf = false, int att = 0) {
    *ok = false;
    if (att && L != 128) return SPL_OK;
    const uint32_t W = L / 32;
    // Private counters cover scores [L/2, L] only: the k-th best agreement is
    // >= L/2 whenever at least k rows agree on half their bits (retrieval
    // keeps a small fraction of the rows); the kernel completes the lower
    // bins from its on-chip scores when that does not hold. Halving the
    // counters is what keeps 3 CTAs/SM under the fast carve-out.
    const uint32_t lo = L / 2;
    const size_t wbins = (size_t)L + 1 - lo;
    if (!vec_ok(codes, stride_rows, W) || wbins * kThreads > 96 * 1024) return SPL_OK;
    const void* fn = nullptr;
    if (L <= 255) {
        switch (W) {
            case 1: fn = shard ? fused_fn<1, uint8_t, true>() : fused_fn<1, uint8_t>(); break;
            case 2: fn = shard ? fused_fn<2, uint8_t, true>() : fused_fn<2, uint8_t>(); break;
            case 4:
                // the decode-step kernels attend their rows themselves: no
                // L2 prefetch in the select (PF = false keeps its loop small)
                if (att == 1)
                    fn = shard ? fused_fn<4, uint8_t, true, false, true, __nv_bfloat16>()
                               : fused_fn<4, uint8_t, false, false, true, __nv_bfloat16>();
                else if (att == 2)
                    fn = shard ? fused_fn<4, uint8_t, true, false, true, float>()
                               : fused_fn<4, uint8_t, false, false, true, float>();
                else
                    fn = shard ? fused_fn<4, uint8_t, true>()
                               : (pf ? fused_fn<4, uint8_t, false, true>() : fused_fn<4, uint8_t>());
                break;
            default: return SPL_OK;
        }
    } else if (shard) {
        return SPL_OK;  // the fused sharded path keeps u8 scores (L <= 255)
    } else if (W == 8) {
        fn = fused_fn<8, uint16_t>();
    } else {
        return SPL_OK;
    }
    const size_t sb = L <= 255 ? 1 : 2;
    const uint64_t total = (uint64_t)P * n_max;
    const size_t base = std::max<size_t>(align_up(wbins * kThreads, 16), K3_SEL_SCRATCH_BYTES) +
                        2 * align_up((size_t)(L + 2) * 4, 16);
    int dev_max_smem = 0, sm_smem = 0;
    SPL_CUDA_TRY(ctx, cudaDeviceGetAttribute(&dev_max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin,
                                             ctx->device));
    SPL_CUDA_TRY(ctx, cudaDeviceGetAttribute(&sm_smem, cudaDevAttrMaxSharedMemoryPerMultiprocessor,
                                             ctx->device));
    // first choice: the most CTAs per SM that stay under the fast carve-out;
    // else the most that fit at all
    for (int pass = 0; pass < 2; ++pass)
    for (int cps = 3; cps >= 1; --cps) {
        const uint64_t G_target = (uint64_t)ctx->num_sms * cps;
        // P <= G_target: a whole number of segments per problem (a CTA whose
        // segment straddled two problems paid a second pipeline ramp, flush
        // and record: ~5 us on the slowest CTA); else equal cuts of P x n_max
        uint64_t S, pstride;
        if (P <= G_target) {
            const uint64_t cpp = G_target / P;
            S = align_up(std::max<uint64_t>((n_max + cpp - 1) / cpp, 1024), 256);
            pstride = align_up(n_max, S);
        } else {
            S = align_up(std::max<uint64_t>((total + G_target - 1) / G_target, 1024), 256);
            pstride = n_max;
        }
        const uint64_t vtotal = (uint64_t)P * pstride;
        const uint64_t pieces = S / pstride + 2;
        const size_t region = align_up((size_t)(S + 16 * pieces) * sb + 16 * pieces, 16);
        const size_t smem = base + region;
        if (smem > (size_t)dev_max_smem || (smem + 1024 + 256) * cps > (size_t)sm_smem) continue;
        if (pass == 0 && (smem + 1024) * cps > kFastCarveBytes) continue;
        SPL_CUDA_TRY(ctx, cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        int per_sm = 0;
        SPL_CUDA_TRY(ctx, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kThreads, smem));
        const uint64_t G = (vtotal + S - 1) / S;
        if ((uint64_t)per_sm * ctx->num_sms < G) continue;
        K3Plan& pl = out->pl;
        pl = K3Plan{};
        pl.vec = true;
        pl.priv = true;
        pl.score_bytes = sb;
        pl.hist_lo = lo;
        pl.g.n_max = n_max;
        pl.g.pstride = pstride;
        pl.g.total = vtotal;
        pl.g.S = S;
        pl.g.G = (uint32_t)G;
        pl.g.P = P;
        pl.g.n_pad = align_up(n_max, 64);
        out->smem = smem;
        out->fn = fn;
        *ok = true;
        return SPL_OK;
    }
    return SPL_OK;
}

// Persistent zeroed per-problem state (self-resetting after every launch):
// [2 sync][counters P][tot P x (L+2)][bar P x 4: fused low-bin fallback counters]
struct K3State {
    uint32_t* sync;
    uint32_t* counters;
    uint32_t* tot;
    uint32_t* bar;
};

spl_status k3_state(spl_ctx* ctx, uint32_t P, uint32_t L, cudaStream_t s, K3State* st) {
    const size_t words = 2 + (size_t)P * (1 + (L + 2) + 4);
    size_t have = ctx->k3_state_words * 4;
    spl_status e = ensure_buffer(ctx, reinterpret_cast<void**>(&ctx->k3_state), &have, words * 4,
                                 true, s, "hamming_topk");
    if (e) return e;
    ctx->k3_state_words = have / 4;
    st->sync = ctx->k3_state;
    st->counters = ctx->k3_state + 2;
    st->tot = st->counters + P;
    st->bar = st->tot + (size_t)P * (L + 2);
    return SPL_OK;
}

struct K3Ws {
    void* scores;
    uint32_t* records;
    uint4* plans;
};

spl_status k3_workspace(spl_ctx* ctx, const K3Plan& pl, uint32_t L, cudaStream_t s, K3Ws* ws,
                        bool global_scores = true) {
    const size_t sc = global_scores ? align_up((size_t)pl.g.P * pl.g.n_pad * pl.score_bytes, 256) : 0;
    const size_t rec = align_up((size_t)(pl.g.G + pl.g.P) * (L + 2) * 4, 256);
    const size_t plans = align_up((size_t)(pl.g.G + pl.g.P) * 16, 256);
    spl_status st = ensure_buffer(ctx, &ctx->k3_ws, &ctx->k3_ws_bytes, sc + rec + plans, false, s,
                                  "hamming_topk");
    if (st) return st;
    uint8_t* b = static_cast<uint8_t*>(ctx->k3_ws);
    ws->scores = b;
    ws->records = reinterpret_cast<uint32_t*>(b + sc);
    ws->plans = reinterpret_cast<uint4*>(b + sc + rec);
    return SPL_OK;
}

spl_status validate_common(spl_ctx* ctx, const char* who, const uint32_t* codes,
                           const uint32_t* qcodes, const uint32_t* n_valid, uint32_t L,
                           uint32_t nvalid_div) {
    if (!ctx) return SPL_E_STATE;
    if (L == 0 || L % 32 != 0 || L > (1u << 15))
        return fail(ctx, SPL_E_DIMENSION,
                    std::string(who) + ": length_bits " + std::to_string(L) +
                        " must be a positive multiple of 32 (at most 32768)");
    if (nvalid_div == 0) return fail(ctx, SPL_E_DIMENSION, std::string(who) + ": nvalid_div == 0");
    if (!codes || !qcodes || !n_valid)
        return fail(ctx, SPL_E_STATE, std::string(who) + ": null device pointer");
    return SPL_OK;
}

spl_status launch_scan(spl_ctx* ctx, const K3Plan& pl, const K3Params& prm, cudaStream_t s) {
    const void* fn = pick_scan(pl, prm.L);
    void* args[] = {const_cast<K3Params*>(&prm)};
    SPL_CUDA_TRY(ctx, launch_pdl(fn, dim3(pl.grid), dim3(kThreads), pl.smem, s, args));
    return after_launch(ctx, "k3_scan");
}

spl_status launch_select(spl_ctx* ctx, const K3Plan& pl, const K3Params& prm, uint32_t* idx,
                         uint64_t idx_stride, cudaStream_t s) {
    const void* fn = pl.score_bytes == 1 ? reinterpret_cast<const void*>(&k3_select<uint8_t>)
                                         : reinterpret_cast<const void*>(&k3_select<uint16_t>);
    K3Params p2 = prm;
    void* args[] = {&p2, &idx, &idx_stride};
    SPL_CUDA_TRY(ctx, launch_pdl(fn, dim3(pl.g.G), dim3(kThreads), 0, s, args));
    return after_launch(ctx, "k3_select");
}

K3Params base_params(spl_ctx* ctx, const K3Plan& pl, const K3Ws& ws, const K3State& kst,
                     const uint32_t* codes, uint64_t stride_rows, uint32_t L,
                     const uint32_t* qcodes, const uint32_t* n_valid, uint32_t nvalid_div,
                     uint32_t k) {
    K3Params prm{};
    prm.codes = codes;
    prm.stride_rows = stride_rows;
    prm.qcodes = qcodes;
    prm.n_valid = n_valid;
    prm.nvalid_div = nvalid_div;
    prm.L = L;
    prm.W = L / 32;
    prm.k = k;
    prm.g = pl.g;
    prm.scores = ws.scores;
    prm.records = ws.records;
    prm.tot_hist = kst.tot;
    prm.tot_stride = L + 2;
    prm.counters = kst.counters;
    prm.sync = kst.sync;
    prm.plans = ws.plans;
    prm.dev_err = ctx->dev_err;
    return prm;
}

void k3_trace_report(uint64_t* dtrace, uint32_t G, uint64_t S, cudaStream_t s) {
    const char* tr = getenv("SPL_K3_TRACE");
    {
                // stamps per CTA (16 slots): 0 start, 1 stream end, 2 past
                // griddepcontrol.wait, 3 T known, 4 prefix, 5 end, 6 smid, 7 attention
                // start (decode step), 8 own record read, 9 select counts, 10 select
                // scan, 11 select emitted
                constexpr int kSlots = 16;
                constexpr int kCols = 11;
                const int cols[kCols] = {0, 2, 1, 3, 4, 8, 9, 10, 11, 7, 5};
                const char* names = "start waited stream thresh prefix rec counts scan emit attend end";
                std::vector<uint64_t> h((size_t)G * kSlots);
                cudaStreamSynchronize(s);
                cudaMemcpy(h.data(), dtrace, h.size() * 8, cudaMemcpyDeviceToHost);
                cudaFree(dtrace);
                uint64_t t0 = ~0ull;
                for (uint32_t i = 0; i < G; ++i) t0 = std::min(t0, h[i * kSlots]);
                double mx[kCols] = {0}, mean[kCols] = {0};
                for (uint32_t i = 0; i < G; ++i)
                    for (int j = 0; j < kCols; ++j) {
                        const uint64_t raw = h[i * kSlots + cols[j]];
                        const double v = raw ? (double)(raw - t0) / 1000.0 : 0.0;
                        mx[j] = std::max(mx[j], v);
                        mean[j] += v / G;
                    }
                fprintf(stderr, "k3_fused trace G=%u S=%llu [%s] mean:", G,
                        (unsigned long long)S, names);
                for (int j = 0; j < kCols; ++j) fprintf(stderr, " %.1f", mean[j]);
                fprintf(stderr, "  max:");
                for (int j = 0; j < kCols; ++j) fprintf(stderr, " %.1f", mx[j]);
                fprintf(stderr, " us");
                double cyc[3] = {0, 0, 0};
                for (uint32_t i = 0; i < G; ++i)
                    for (int j = 0; j < 3; ++j)
                        cyc[j] += (double)(int64_t)(h[i * kSlots + 13 + j] - h[i * kSlots + 12 + j]) / G;
                fprintf(stderr, "  select thread-0 cycles: counts %.0f scan %.0f emit %.0f\n", cyc[0], cyc[1],
                        cyc[2]);
                if (*tr == '2') {  // per-CTA dump: cta, smid, stamps (us)
                    const char* path = getenv("SPL_K3_TRACE_CSV");
                    FILE* f = fopen(path && *path ? path : "gpurun_out/k3_trace.csv", "w");
                    if (!f) fprintf(stderr, "k3 trace: cannot write %s\n", path ? path : "gpurun_out/k3_trace.csv");
                    if (f) {
                        fprintf(f, "cta,smid,start,waited,stream,thresh,prefix,rec,counts,scan,emit,attend,end\n");
                        for (uint32_t i = 0; i < G; ++i) {
                            fprintf(f, "%u,%llu", i, (unsigned long long)h[i * kSlots + 6]);
                            for (int j = 0; j < kCols; ++j) {
                                const uint64_t raw = h[i * kSlots + cols[j]];
                                fprintf(f, ",%.3f", raw ? (double)(raw - t0) / 1000.0 : 0.0);
                            }
                            fprintf(f, "\n");
                        }
                        fclose(f);
                    }
                }
            }
}

// Cooperative launch of the fused kernels: SM-limited contexts (detected at
// spl_ctx_create) or SPL_K3_COOP=1 (read per call).
bool k3_coop(const spl_ctx* ctx) {
    if (ctx->k3_coop) return true;
    const char* e = getenv("SPL_K3_COOP");
    return e && *e == '1';
}

// SPL_K3_PATH=twopass forces the two-kernel path (A/B measurement, tests).
bool fused_allowed() {
    const char* e = getenv("SPL_K3_PATH");
    return !(e && std::string(e) == "twopass");
}

}  // namespace

spl_status hamming_topk_impl(spl_ctx* ctx, const uint32_t* codes, uint64_t stride_rows,
                             uint32_t L, const uint32_t* qcodes, uint32_t P,
                             const uint32_t* n_valid, uint32_t nvalid_div, uint64_t n_max,
                             uint32_t k, uint32_t* idx, uint32_t* cnt, cudaStream_t s) {
    spl_status st = validate_common(ctx, "hamming_topk", codes, qcodes, n_valid, L, nvalid_div);
    if (st) return st;
    if (k == 0) return fail(ctx, SPL_E_DIMENSION, "hash_topk: k must be >= 1");
    if (!idx || !cnt) return fail(ctx, SPL_E_STATE, "hamming_topk: null output pointer");
    if (P == 0) return SPL_OK;
    if (n_max == 0) {
        SPL_CUDA_TRY(ctx, cudaMemsetAsync(cnt, 0, sizeof(uint32_t) * P, s));
        return SPL_OK;
    }
    if (n_max > 0xFFFFFFFFull) return fail(ctx, SPL_E_DIMENSION, "hamming_topk: n_max exceeds 2^32 rows");
    if (stride_rows != 0 && n_max > stride_rows)
        return fail(ctx, SPL_E_DIMENSION,
                    "hamming_topk: n_max=" + std::to_string(n_max) + " exceeds the problem stride of " +
                        std::to_string(stride_rows) + " rows");
    K3State kst;
    if ((st = k3_state(ctx, P, L, s, &kst))) return st;
    if (fused_allowed()) {
        bool ok = false;
        K3FPlan fp{};
        // the decode step's prefetching variant (select warms L2 for K4) is a
        // separate instantiation: the plain retrieval kernel carries no trace of it
        const bool pf = ctx->k3_pf_k != nullptr;
        if ((st = make_fused_plan(ctx, P, n_max, L, codes, stride_rows, &ok, &fp, false, pf))) return st;
        if (ok) {
            K3Ws ws;
            if ((st = k3_workspace(ctx, fp.pl, L, s, &ws, false))) return st;
            K3Params prm =
                base_params(ctx, fp.pl, ws, kst, codes, stride_rows, L, qcodes, n_valid, nvalid_div, k);
            prm.cnt_out = cnt;
            prm.idx_out = idx;
            prm.pf_k = static_cast<const char*>(ctx->k3_pf_k);
            prm.pf_v = static_cast<const char*>(ctx->k3_pf_v);
            prm.pf_row_bytes = ctx->k3_pf_row_bytes;
            prm.idx_stride = k;
            prm.hist_lo = fp.pl.hist_lo;
            prm.counters2 = kst.bar;
            const uint32_t G = fp.pl.g.G;
            const char* tr = getenv("SPL_K3_TRACE");
            uint64_t* dtrace = nullptr;
            if (tr && *tr && !stream_capturing(s)) {
                SPL_CUDA_TRY(ctx, cudaMalloc(&dtrace, (size_t)G * 16 * 8));
                SPL_CUDA_TRY(ctx, cudaMemsetAsync(dtrace, 0, (size_t)G * 16 * 8, s));
            }
            prm.trace = dtrace;
            void* args[] = {&prm};
            bool launched = true;
            if (k3_coop(ctx)) {
                // cooperative: co-residency guaranteed by the driver, or the
                // launch is refused and the two-pass kernels below run instead
                const cudaError_t e = cudaLaunchCooperativeKernel(fp.fn, dim3(G), dim3(kThreads), args, fp.smem, s);
                if (e == cudaErrorCooperativeLaunchTooLarge) {
                    cudaGetLastError();
                    launched = false;
                } else {
                    SPL_CUDA_TRY(ctx, e);
                }
            } else {
                SPL_CUDA_TRY(ctx, launch_pdl(fp.fn, dim3(G), dim3(kThreads), fp.smem, s, args));
            }
            if (!launched) {
                if (dtrace) cudaFree(dtrace);
            } else {
            st = after_launch(ctx, pf ? "k3_fused_pf" : "k3_fused");
            if (dtrace) k3_trace_report(dtrace, G, fp.pl.g.S, s);
            return st;
            }
        }
    }
    K3Plan pl;
    if ((st = make_plan(ctx, P, n_max, L, codes, stride_rows, &pl, true))) return st;
    K3Ws ws;
    if ((st = k3_workspace(ctx, pl, L, s, &ws))) return st;
    K3Params prm = base_params(ctx, pl, ws, kst, codes, stride_rows, L, qcodes, n_valid, nvalid_div, k);
    prm.cnt_out = cnt;
    prm.idx_out = idx;
    prm.idx_stride = k;
    prm.shard = 0;
    prm.hist_lo = pl.hist_lo;
    prm.clamp8 = pl.clamp8 ? 1 : 0;
    // SPL_K3_TIME=1: print the two-pass kernels' device times (diagnostics)
    const char* tm = getenv("SPL_K3_TIME");
    cudaEvent_t ev[3];
    const bool timed = tm && *tm == '1' && !stream_capturing(s);
    if (timed) {
        for (auto& e : ev) cudaEventCreate(&e);
        cudaEventRecord(ev[0], s);
    }
    if ((st = launch_scan(ctx, pl, prm, s))) return st;
    if (timed) cudaEventRecord(ev[1], s);
    st = launch_select(ctx, pl, prm, idx, k, s);
    if (timed) {
        cudaEventRecord(ev[2], s);
        cudaEventSynchronize(ev[2]);
        float a = 0, b = 0;
        cudaEventElapsedTime(&a, ev[0], ev[1]);
        cudaEventElapsedTime(&b, ev[1], ev[2]);
        fprintf(stderr, "k3 two-pass: scan %.1f us (G=%u grid=%u S=%llu), select %.1f us\n", a * 1e3,
                pl.g.G, pl.grid, (unsigned long long)pl.g.S, b * 1e3);
        for (auto& e : ev) cudaEventDestroy(e);
    }
    return st;
}

// Decode-step retrieval + attention in ONE launch (k3_fused<.., ATT>): same
// indices as hamming_topk_impl, plus out[p] = sparse attention of q[p] over
// the selected rows U {own}. *done = false (and nothing launched) when the
// fused geometry does not apply (L != 128, d != 128, scores too large for
// shared memory, SPL_K3_PATH=twopass): the caller then runs K3 + K4.
// peer != nullptr: one rank of a sequence-sharded cache (k3_fused<SHARD,
// ATT>): histograms and then the per-problem partial attention are exchanged
// with the other ranks inside the kernel; idx / cnt / out_offset are this
// rank's share (as spl_hamming_topk_sharded), out the full result on every
// rank; own != 0 on the rank that holds the own row (its local n_valid - 1).
spl_status hamming_topk_attend_impl(spl_ctx* ctx, const uint32_t* codes, uint64_t stride_rows,
                                    uint32_t L, const uint32_t* qcodes, uint32_t P,
                                    const uint32_t* n_valid, uint32_t nvalid_div, uint64_t n_max,
                                    uint32_t k, uint32_t* idx, uint32_t* cnt, const float* q,
                                    const void* kcache, const void* vcache, int kv_dtype, uint32_t d,
                                    float qscale, float* out, cudaStream_t s, bool* done,
                                    spl_peer* peer, uint32_t* out_offset, int own) {
    *done = false;
    if (peer && (!peer->connected || P > peer->Pmax || L > peer->Lmax ||
                 (size_t)peer->R * (L + 2) * 4 > K3_SEL_SCRATCH_BYTES))
        return SPL_OK;
    if (d != 128 || L != 128 || (kv_dtype != SPL_BF16 && kv_dtype != SPL_F32) || !fused_allowed())
        return SPL_OK;
    const char* e = getenv("SPL_DECODE_FUSED");
    if (e && *e == '0') return SPL_OK;
    spl_status st = validate_common(ctx, "hamming_topk", codes, qcodes, n_valid, L, nvalid_div);
    if (st) return st;
    if (k == 0) return fail(ctx, SPL_E_DIMENSION, "hash_topk: k must be >= 1");
    if (P == 0 || n_max == 0 || n_max > 0xFFFFFFFFull) return SPL_OK;
    if (stride_rows == 0 || n_max > stride_rows) return SPL_OK;
    bool ok = false;
    K3FPlan fp{};
    if ((st = make_fused_plan(ctx, P, n_max, L, codes, stride_rows, &ok, &fp, peer != nullptr, true,
                              kv_dtype == SPL_BF16 ? 1 : 2)))
        return st;
    if (!ok) return SPL_OK;
    K3State kst;
    if ((st = k3_state(ctx, P, L, s, &kst))) return st;
    K3Ws ws;
    if ((st = k3_workspace(ctx, fp.pl, L, s, &ws, false))) return st;
    const uint32_t G = fp.pl.g.G;
    if ((st = ensure_buffer(ctx, reinterpret_cast<void**>(&ctx->att_ws), &ctx->att_ws_bytes,
                            (size_t)(G + P) * (d + 2) * sizeof(float), false, s, "decode_step")))
        return st;
    size_t have = ctx->att_counters_n * 4;
    if ((st = ensure_buffer(ctx, reinterpret_cast<void**>(&ctx->att_counters), &have, (size_t)P * 4,
                            true, s, "decode_step")))
        return st;
    ctx->att_counters_n = have / 4;
    K3Params prm = base_params(ctx, fp.pl, ws, kst, codes, stride_rows, L, qcodes, n_valid, nvalid_div, k);
    prm.cnt_out = cnt;
    prm.idx_out = idx;
    prm.idx_stride = k;
    prm.hist_lo = fp.pl.hist_lo;
    prm.counters2 = kst.bar;
    const uint32_t row_bytes = d * (kv_dtype == SPL_BF16 ? 2u : 4u);
    prm.pf_k = static_cast<const char*>(kcache);
    prm.pf_v = static_cast<const char*>(vcache);
    prm.pf_row_bytes = row_bytes;
    prm.att_q = q;
    prm.att_qscale = qscale;
    prm.att_part = ctx->att_ws;
    prm.att_cnt = ctx->att_counters;
    prm.att_out = out;
    prm.att_own = peer ? (own ? 1 : 0) : 1;
    if (peer) {
        prm.peer_bufs = peer->d_table;
        prm.own_buf = peer->buf;
        prm.R = peer->R;
        prm.rank = peer->rank;
        prm.Pmax = peer->Pmax;
        prm.epoch_ptr = peer->d_epoch;
        prm.out_offset = out_offset;
        prm.part_off = (uint32_t)xwords(peer->R, peer->Pmax, peer->Lmax + 2);
    }
    const char* tr = getenv("SPL_K3_TRACE");
    uint64_t* dtrace = nullptr;
    if (tr && *tr && !stream_capturing(s)) {
        SPL_CUDA_TRY(ctx, cudaMalloc(&dtrace, (size_t)G * 16 * 8));
        SPL_CUDA_TRY(ctx, cudaMemsetAsync(dtrace, 0, (size_t)G * 16 * 8, s));
    }
    prm.trace = dtrace;
    void* args[] = {&prm};
    if (k3_coop(ctx)) {
        const cudaError_t e = cudaLaunchCooperativeKernel(fp.fn, dim3(G), dim3(kThreads), args, fp.smem, s);
        if (e == cudaErrorCooperativeLaunchTooLarge && !peer) {
            // the unfused decode step (K3 then K4) runs instead
            cudaGetLastError();
            if (dtrace) cudaFree(dtrace);
            return SPL_OK;
        }
        SPL_CUDA_TRY(ctx, e);
    } else {
        SPL_CUDA_TRY(ctx, launch_pdl(fp.fn, dim3(G), dim3(kThreads), fp.smem, s, args));
    }
    if ((st = after_launch(ctx, peer ? "k3_fused_shard_attend" : "k3_fused_attend"))) return st;
    if (dtrace) k3_trace_report(dtrace, G, fp.pl.g.S, s);
    *done = true;
    return SPL_OK;
}

spl_status peer_combine_launch(spl_ctx* ctx, spl_peer* peer, const float* partials, uint32_t P,
                               uint32_t d, float* out, cudaStream_t s) {
    if (!peer || !peer->connected) return fail(ctx, SPL_E_STATE, "peer_combine: peer group not connected");
    if (d == 0 || d > kPartDMax)
        return fail(ctx, SPL_E_DIMENSION, "sharded_decode_step: head dim must be 1 .. 256");
    if (P == 0) return SPL_OK;
    K3Params prm{};
    prm.peer_bufs = peer->d_table;
    prm.own_buf = peer->buf;
    prm.R = peer->R;
    prm.rank = peer->rank;
    prm.Pmax = peer->Pmax;
    prm.epoch_ptr = peer->d_epoch;
    prm.part_off = (uint32_t)xwords(peer->R, peer->Pmax, peer->Lmax + 2);
    prm.dev_err = ctx->dev_err;
    k5_peer_combine<<<P, (d + 31) / 32 * 32, 0, s>>>(prm, partials, d, out);
    return after_launch(ctx, "k5_peer_combine");
}

spl_status shard_histogram_impl(spl_ctx* ctx, const uint32_t* codes, uint64_t stride_rows,
                                uint32_t L, const uint32_t* qcodes, uint32_t P,
                                const uint32_t* n_valid, uint32_t nvalid_div, uint64_t n_max,
                                uint32_t* hist, cudaStream_t s) {
    spl_status st = validate_common(ctx, "shard_histogram", codes, qcodes, n_valid, L, nvalid_div);
    if (st) return st;
    if (!hist) return fail(ctx, SPL_E_STATE, "shard_histogram: null hist");
    SPL_CUDA_TRY(ctx, cudaMemsetAsync(hist, 0, sizeof(uint32_t) * P * (L + 1), s));
    ctx->shard_n_max = n_max;
    ctx->shard_P = P;
    ctx->shard_L = L;
    if (P == 0 || n_max == 0) {
        ctx->shard_G = 0;
        return SPL_OK;
    }
    K3Plan pl;
    if ((st = make_plan(ctx, P, n_max, L, codes, stride_rows, &pl))) return st;
    K3Ws ws;
    if ((st = k3_workspace(ctx, pl, L, s, &ws))) return st;
    K3State kst;
    if ((st = k3_state(ctx, P, L, s, &kst))) return st;
    ctx->shard_G = pl.g.G;
    ctx->shard_S = pl.g.S;
    K3Params prm = base_params(ctx, pl, ws, kst, codes, stride_rows, L, qcodes, n_valid, nvalid_div, 1);
    prm.tot_hist = hist;
    prm.tot_stride = L + 1;
    prm.shard = 1;
    return launch_scan(ctx, pl, prm, s);
}

spl_status shard_select_impl(spl_ctx* ctx, const uint32_t* all_hist, uint32_t R, uint32_t rank,
                             uint32_t L, uint32_t P, const uint32_t* n_valid, uint32_t nvalid_div,
                             uint64_t n_max, uint32_t k, uint32_t* idx, uint32_t* cnt,
                             uint32_t* out_offset, cudaStream_t s) {
    if (!ctx) return SPL_E_STATE;
    if (k == 0) return fail(ctx, SPL_E_DIMENSION, "hash_topk: k must be >= 1");
    if (R == 0 || rank >= R) return fail(ctx, SPL_E_DIMENSION, "shard_select: rank out of range");
    if (ctx->shard_P != P || ctx->shard_L != L || ctx->shard_n_max != n_max)
        return fail(ctx, SPL_E_STATE,
                    "shard_select: geometry differs from the preceding shard_histogram");
    if (P == 0) return SPL_OK;
    if (n_max == 0)
        return fail(ctx, SPL_E_DIMENSION, "shard_select: every rank must own at least one row");
    // the select phase must cut rows exactly like the preceding histogram
    K3Plan pl{};
    spl_status st;
    pl.g.n_max = n_max;
    pl.g.pstride = n_max;
    pl.g.total = (uint64_t)P * n_max;
    pl.g.S = ctx->shard_S;
    pl.g.G = ctx->shard_G;
    pl.g.P = P;
    pl.g.n_pad = align_up(n_max, 64);
    pl.score_bytes = L <= 255 ? 1 : 2;
    K3Ws ws;
    if ((st = k3_workspace(ctx, pl, L, s, &ws))) return st;
    K3State kst;
    if ((st = k3_state(ctx, P, L, s, &kst))) return st;
    K3Params prm = base_params(ctx, pl, ws, kst, nullptr, 0, L, nullptr, n_valid, nvalid_div, k);
    prm.cnt_out = cnt;
    prm.shard = 1;
    const size_t plan_smem = (size_t)(L + 2) * 4;
    if (plan_smem > 48 * 1024)
        SPL_CUDA_TRY(ctx, cudaFuncSetAttribute(k3_shard_plan, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                               (int)plan_smem));
    k3_shard_plan<<<P, kThreads, plan_smem, s>>>(prm, all_hist, R, rank, out_offset);
    if ((st = after_launch(ctx, "k3_shard_plan"))) return st;
    return launch_select(ctx, pl, prm, idx, k, s);
}

uint64_t peer_area_words(uint32_t R, uint32_t Pmax, uint32_t Lmax) {
    return xwords(R, Pmax, Lmax + 2) + part_words(R, Pmax);  // histograms + partials
}

// ------------------------------------------------ fused sharded retrieval
spl_status hamming_topk_sharded_impl(spl_ctx* ctx, spl_peer* peer, const uint32_t* codes,
                                     uint64_t stride_rows, uint32_t L, const uint32_t* qcodes,
                                     uint32_t P, const uint32_t* n_valid, uint32_t nvalid_div,
                                     uint64_t n_max, uint32_t k, uint32_t* idx, uint32_t* cnt,
                                     uint32_t* out_offset, cudaStream_t s) {
    spl_status st = validate_common(ctx, "hamming_topk_sharded", codes, qcodes, n_valid, L, nvalid_div);
    if (st) return st;
    if (!peer || !peer->connected) return fail(ctx, SPL_E_STATE, "hamming_topk_sharded: peer group not connected");
    if (k == 0) return fail(ctx, SPL_E_DIMENSION, "hash_topk: k must be >= 1");
    if (!idx || !cnt || !out_offset) return fail(ctx, SPL_E_STATE, "hamming_topk_sharded: null output pointer");
    if (P > peer->Pmax || L > peer->Lmax)
        return fail(ctx, SPL_E_DIMENSION, "hamming_topk_sharded: P or L exceeds the peer group's capacity");
    if (P == 0) return SPL_OK;
    if (n_max == 0 || n_max > 0xFFFFFFFFull)
        return fail(ctx, SPL_E_DIMENSION, "hamming_topk_sharded: every rank must own 1 .. 2^32 rows");
    K3State kst;
    if ((st = k3_state(ctx, P, L, s, &kst))) return st;
    bool ok = false;
    K3FPlan fp{};
    if ((st = make_fused_plan(ctx, P, n_max, L, codes, stride_rows, &ok, &fp, true))) return st;
    if (!ok || (size_t)peer->R * (L + 2) * 4 > K3_SEL_SCRATCH_BYTES)
        return fail(ctx, SPL_E_STATE,
                    "hamming_topk_sharded: the local cache (or R x (L + 2) histogram words) does not "
                    "fit the fused path; use spl_shard_histogram + collective + spl_shard_select");
    K3Ws ws;
    if ((st = k3_workspace(ctx, fp.pl, L, s, &ws, false))) return st;
    K3Params prm = base_params(ctx, fp.pl, ws, kst, codes, stride_rows, L, qcodes, n_valid, nvalid_div, k);
    prm.cnt_out = cnt;
    prm.idx_out = idx;
    prm.idx_stride = k;
    prm.hist_lo = fp.pl.hist_lo;
    prm.counters2 = kst.bar;
    prm.peer_bufs = peer->d_table;
    prm.own_buf = peer->buf;
    prm.R = peer->R;
    prm.rank = peer->rank;
    prm.Pmax = peer->Pmax;
    prm.epoch_ptr = peer->d_epoch;
    prm.out_offset = out_offset;
    const char* tr = getenv("SPL_K3_TRACE");
    uint64_t* dtrace = nullptr;
    if (tr && *tr && !stream_capturing(s)) {
        SPL_CUDA_TRY(ctx, cudaMalloc(&dtrace, (size_t)fp.pl.g.G * 16 * 8));
        SPL_CUDA_TRY(ctx, cudaMemsetAsync(dtrace, 0, (size_t)fp.pl.g.G * 16 * 8, s));
    }
    prm.trace = dtrace;
    void* args[] = {&prm};
    if (k3_coop(ctx))
        SPL_CUDA_TRY(ctx, cudaLaunchCooperativeKernel(fp.fn, dim3(fp.pl.g.G), dim3(kThreads), args, fp.smem, s));
    else
        SPL_CUDA_TRY(ctx, cudaLaunchKernel(fp.fn, dim3(fp.pl.g.G), dim3(kThreads), args, fp.smem, s));
    st = after_launch(ctx, "k3_fused_shard");
    if (dtrace) k3_trace_report(dtrace, fp.pl.g.G, fp.pl.g.S, s);
    return st;
}

// Force the lazy load of the sharded-path kernels (see encode_preload): a
// peer group's kernels wait for each other inside, so no member may hit a
// module load (a context synchronisation) in the middle of a step.
void k3_preload() {
    cudaFuncAttributes a;
    const void* fns[] = {fused_fn<1, uint8_t, true>(), fused_fn<2, uint8_t, true>(),
                         fused_fn<4, uint8_t, true>(),
                         fused_fn<4, uint8_t, true, true, true, __nv_bfloat16>(),
                         fused_fn<4, uint8_t, true, true, true, float>(),
                         reinterpret_cast<const void*>(&k5_peer_combine)};
    for (const void* f : fns) cudaFuncGetAttributes(&a, f);
}

}  // namespace spl

extern "C" spl_status spl_plan_shard_host(const uint32_t* all_hist, uint32_t R, uint32_t rank,
                                          uint32_t L, uint32_t k, uint32_t* T, uint32_t* quota,
                                          uint32_t* take_eq, uint32_t* count, uint32_t* offset) {
    if (!all_hist || R == 0 || rank >= R) return SPL_E_DIMENSION;
    const spl_shard_plan p = spl_plan_shard(all_hist, (uint64_t)L + 1, R, rank, L, k);
    if (T) *T = p.T;
    if (quota) *quota = p.quota;
    if (take_eq) *take_eq = p.take_eq;
    if (count) *count = p.T == SPL_PLAN_SKIP ? 0 : p.count;
    if (offset) *offset = p.offset;
    return SPL_OK;
}
