// K3 — HBM-streaming Hamming scan + bit-exact top-k select (sm_100a).
//
// Replaces nxor_scores_into (bitcodes.cpp:59-76) + top_k_indices<int32_t>
// (bitcodes.cpp:89-131) as hash_topk composes them (attention_eval.cpp:
// 172-179), batched over P (batch, head) problems.
//
// Layout: codes [P][stride][W] u32 (row = one 16 B / 32 B vector for
// L = 128 / 256). The virtual row space P x n_max is cut into G equal
// contiguous CTA ranges (G = SMs x resident CTAs, one wave, no tail); a
// CTA's range is split at problem boundaries into "segments" (record index
// cta + problem, unique because the (cta, problem) staircase is monotone).
//
// k3_scan   : per row score = L - sum popc(q ^ r) from 128-bit streaming
//             loads (L2 evict-first), u8/u16 score to an L2-resident buffer,
//             per-thread private u16 histograms in shared memory (LDS/STS,
//             conflict-free, no atomics — a smem-atomic histogram cannot
//             keep up with ~1.5 rows/clk/SM), reduced per segment to a
//             suffix-cumulative record. The CTA finishing a problem's last
//             segment plans it (T, tie quota, per-segment output offsets).
// k3_select : re-reads the u8 scores (from L2) and does the ordered
//             compaction: score > T, or score == T among the first `take`
//             ties of the segment; output ascending, bit-exact.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <string>

#include "spl_launch.cuh"
#include "spl_plan.cuh"

namespace spl {

struct K3Geom {
    uint64_t n_max;  // rows per problem (virtual)
    uint64_t total;  // P * n_max
    uint64_t S;      // rows per CTA
    uint64_t n_pad;  // score row stride
    uint32_t G;      // CTAs
    uint32_t P;
};

__host__ __device__ __forceinline__ uint32_t seg_first(const K3Geom& g, uint32_t p) {
    return (uint32_t)(((uint64_t)p * g.n_max) / g.S);
}
__host__ __device__ __forceinline__ uint32_t seg_last(const K3Geom& g, uint32_t p) {
    return (uint32_t)((((uint64_t)p + 1) * g.n_max - 1) / g.S);
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
    void* scores;          // [P][n_pad] ScoreT
    uint32_t* records;     // [(G+P)][L+2] suffix-cumulative counts
    uint32_t* tot_hist;    // [P][tot_stride]
    uint64_t tot_stride;
    uint32_t* counters;    // [P]
    uint4* plans;          // [(G+P)] {T, offset, take, 0}
    uint32_t* cnt_out;     // [P]
    uint32_t* dev_err;
    int shard;             // 1: no planning; tot_hist = caller's histogram
};

constexpr int kThreads = 256;

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
    // process from the top in chunks of kThreads, reversed index
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

// Plan every segment of problem p given (T, quota): per segment output
// offset + ties to take, from the segment records (read through L2: they
// were written by other CTAs of this launch).
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
            prm.plans[c + p] = make_uint4(T, off, take, 0u);
        }
        carry_gt += tot & 0xffffffffu;
        carry_eq += tot >> 32;
    }
}

// Single-GPU planning by the CTA that completed problem p's last segment.
__device__ void plan_problem_single(const K3Params& prm, uint32_t p, uint32_t nv,
                                    uint32_t* s_cum, uint64_t* s_warp, uint32_t* s_T) {
    const uint32_t L = prm.L;
    uint32_t* tot = prm.tot_hist + (uint64_t)p * prm.tot_stride;
    for (uint32_t t = threadIdx.x; t <= L + 1; t += kThreads) {
        s_cum[t] = t <= L ? __ldcg(tot + t) : 0u;
        if (t <= L) tot[t] = 0u;  // self-reset for the next launch
    }
    __syncthreads();
    block_suffix_sum(s_cum, L + 1, s_warp);
    const uint32_t kk = prm.k < nv ? prm.k : nv;
    if (threadIdx.x == 0) *s_T = SPL_PLAN_SKIP;
    __syncthreads();
    if (kk > 0) {
        for (uint32_t t = threadIdx.x; t <= L; t += kThreads)
            if (s_cum[t] >= kk && s_cum[t + 1] < kk) *s_T = t;
    }
    __syncthreads();
    const uint32_t T = *s_T;
    const uint32_t quota = (T == SPL_PLAN_SKIP) ? 0u : kk - s_cum[T + 1];
    plan_segments(prm, p, T, quota, s_warp);
    if (threadIdx.x == 0) {
        prm.cnt_out[p] = kk;
        prm.counters[p] = 0u;
    }
}

// ------------------------------------------------------------------ scan
// One 32-byte unit per thread per load (LDG.E.NA.EFL2.256: 256-bit,
// no L1 allocation, L2 evict-first) = 8 / W code rows.
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

// HMODE 0: private per-thread u16 histograms [bins][kThreads]
// HMODE 1: one shared u32 histogram with smem atomics (large L)
template <int W, typename ScoreT, int HMODE>
__global__ void __launch_bounds__(kThreads) k3_scan(K3Params prm) {
    extern __shared__ __align__(16) uint8_t smem[];
    __shared__ uint64_t s_warp[kThreads / 32 + 1];
    __shared__ uint32_t s_flag;
    __shared__ uint32_t s_T;
    const uint32_t L = prm.L;
    const uint32_t bins = L + 1;
    const uint32_t Wr = (W > 0) ? (uint32_t)W : prm.W;
    const size_t hist_bytes =
        HMODE == 0 ? (size_t)bins * kThreads * sizeof(uint16_t) : (size_t)bins * sizeof(uint32_t);
    uint16_t* hist16 = reinterpret_cast<uint16_t*>(smem);
    uint32_t* hist32 = reinterpret_cast<uint32_t*>(smem);
    // HMODE 1 reduces in place: the shared histogram becomes the record.
    uint32_t* s_cum = HMODE == 0
                          ? reinterpret_cast<uint32_t*>(smem + ((hist_bytes + 15) & ~size_t(15)))
                          : hist32;
    const int tid = threadIdx.x;
    const K3Geom& g = prm.g;

    const uint64_t g0 = (uint64_t)blockIdx.x * g.S;
    const uint64_t g1 = min(g0 + g.S, g.total);
    for (uint32_t p = (uint32_t)(g0 / g.n_max); p < g.P && (uint64_t)p * g.n_max < g1; ++p) {
        const uint64_t pbase = (uint64_t)p * g.n_max;
        const uint64_t lo = max(g0, pbase) - pbase;
        const uint64_t hi = min(g1, pbase + g.n_max) - pbase;
        uint32_t nv = prm.n_valid[p / prm.nvalid_div];
        if (nv > g.n_max) {
            if (tid == 0) raise_dev_err(prm.dev_err, SPL_DEV_ERR_DIMENSION);
            nv = (uint32_t)g.n_max;
        }
        const uint64_t r0 = lo, r1 = min(hi, (uint64_t)nv);

        // zero the histogram
        if (HMODE == 0) {
            uint4* h4 = reinterpret_cast<uint4*>(hist16);
            for (uint32_t i = tid; i < hist_bytes / 16; i += kThreads) h4[i] = make_uint4(0, 0, 0, 0);
        } else {
            for (uint32_t i = tid; i < bins; i += kThreads) hist32[i] = 0;
        }
        __syncthreads();

        if (r0 < r1) {
            const uint32_t* qp = prm.qcodes + (uint64_t)p * Wr;
            const uint32_t* base = prm.codes + (uint64_t)p * prm.stride_rows * Wr;
            ScoreT* srow = reinterpret_cast<ScoreT*>(prm.scores) + (uint64_t)p * g.n_pad;
            if constexpr (W > 0) {
                constexpr int R = 8 / W;  // rows per 32-byte unit
                uint32_t q[W];
#pragma unroll
                for (int w = 0; w < W; ++w) q[w] = __ldg(qp + w);
                constexpr int U = 4;
                const uint64_t u0 = r0 / R, u1 = (r1 + R - 1) / R;
                for (uint64_t u = u0 + tid; u < u1; u += (uint64_t)kThreads * U) {
                    Unit32 v[U];
#pragma unroll
                    for (int j = 0; j < U; ++j) {
                        const uint64_t uu = u + (uint64_t)j * kThreads;
                        if (uu < u1) v[j].load(base, uu);
                    }
#pragma unroll
                    for (int j = 0; j < U; ++j) {
                        const uint64_t uu = u + (uint64_t)j * kThreads;
                        if (uu >= u1) continue;
                        uint32_t sc[R];
#pragma unroll
                        for (int r = 0; r < R; ++r) {
                            uint32_t mism = 0;
#pragma unroll
                            for (int w = 0; w < W; ++w) mism += __popc(v[j].w[r * W + w] ^ q[w]);
                            sc[r] = L - mism;
                        }
                        const uint64_t row0 = uu * R;
                        if (row0 >= r0 && row0 + R <= r1) {
                            store_scores<ScoreT, R>(srow + row0, sc);
#pragma unroll
                            for (int r = 0; r < R; ++r) {
                                if (HMODE == 0)
                                    hist16[sc[r] * kThreads + tid] += 1;
                                else
                                    atomicAdd(&hist32[sc[r]], 1u);
                            }
                        } else {
#pragma unroll
                            for (int r = 0; r < R; ++r) {
                                const uint64_t row = row0 + r;
                                if (row < r0 || row >= r1) continue;
                                srow[row] = (ScoreT)sc[r];
                                if (HMODE == 0)
                                    hist16[sc[r] * kThreads + tid] += 1;
                                else
                                    atomicAdd(&hist32[sc[r]], 1u);
                            }
                        }
                    }
                }
            } else {
                for (uint64_t r = r0 + tid; r < r1; r += kThreads) {
                    const uint32_t* row = base + r * Wr;
                    uint32_t mism = 0;
                    for (uint32_t w = 0; w < Wr; ++w) mism += __popc(__ldg(row + w) ^ __ldg(qp + w));
                    const uint32_t s = L - mism;
                    srow[r] = (ScoreT)s;
                    if (HMODE == 0)
                        hist16[s * kThreads + tid] += 1;
                    else
                        atomicAdd(&hist32[s], 1u);
                }
            }
        }
        __syncthreads();

        // reduce -> s_cum[b] = count of score b; s_cum[L+1] = 0
        if (HMODE == 0) {
            const int lane = tid & 31, warp = tid >> 5;
            for (uint32_t b = warp; b < bins; b += kThreads / 32) {
                const uint32_t* h32 = reinterpret_cast<const uint32_t*>(hist16 + (size_t)b * kThreads);
                uint32_t sum = 0;
#pragma unroll
                for (int i = 0; i < kThreads / 64; ++i) {
                    const uint32_t x = h32[lane + 32 * i];
                    sum += (x & 0xffffu) + (x >> 16);
                }
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
                if (lane == 0) s_cum[b] = sum;
            }
        }
        if (tid == 0) s_cum[bins] = 0;
        __syncthreads();
        // raw counts -> global per-problem histogram (integer atomics: the
        // sums are order-independent, so results stay deterministic)
        uint32_t* tot = prm.tot_hist + (uint64_t)p * prm.tot_stride;
        for (uint32_t b = tid; b < bins; b += kThreads)
            if (s_cum[b]) atomicAdd(tot + b, s_cum[b]);
        __syncthreads();
        block_suffix_sum(s_cum, bins, s_warp);
        uint32_t* rec = prm.records + (uint64_t)(blockIdx.x + p) * (L + 2);
        for (uint32_t t = tid; t < L + 2; t += kThreads) rec[t] = s_cum[t];

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
                plan_problem_single(prm, p, nv, s_cum, s_warp, &s_T);
            }
        }
        __syncthreads();
    }
}

// ---------------------------------------------------------------- select
template <typename ScoreT>
__global__ void __launch_bounds__(kThreads) k3_select(K3Params prm, uint32_t* idx,
                                                      uint64_t idx_stride) {
    __shared__ uint64_t s_warp[kThreads / 32 + 1];
    constexpr int PER = 16 / sizeof(ScoreT);
    const K3Geom& g = prm.g;
    const int tid = threadIdx.x;
    const uint64_t g0 = (uint64_t)blockIdx.x * g.S;
    const uint64_t g1 = min(g0 + g.S, g.total);
    for (uint32_t p = (uint32_t)(g0 / g.n_max); p < g.P && (uint64_t)p * g.n_max < g1; ++p) {
        const uint64_t pbase = (uint64_t)p * g.n_max;
        const uint64_t lo = max(g0, pbase) - pbase;
        const uint64_t hi = min(g1, pbase + g.n_max) - pbase;
        uint32_t nv = prm.n_valid[p / prm.nvalid_div];
        if (nv > g.n_max) nv = (uint32_t)g.n_max;
        const uint64_t r0 = lo, r1 = min(hi, (uint64_t)nv);
        const uint4 plan = prm.plans[blockIdx.x + p];
        const uint32_t T = plan.x;
        if (T == SPL_PLAN_SKIP || r0 >= r1) continue;  // uniform across the block
        const uint32_t take = plan.z;
        uint32_t* out = idx + (uint64_t)p * idx_stride + plan.y;
        const ScoreT* srow = reinterpret_cast<const ScoreT*>(prm.scores) + (uint64_t)p * g.n_pad;
        uint64_t carry_gt = 0, carry_eq = 0;
        const uint64_t a0 = r0 & ~(uint64_t)(PER - 1);
        for (uint64_t tile = a0; tile < r1; tile += (uint64_t)kThreads * PER) {
            const uint64_t my = tile + (uint64_t)tid * PER;
            ScoreT s[PER];
            if (my < r1) {
                const uint4 v = *reinterpret_cast<const uint4*>(srow + my);
                const ScoreT* sv = reinterpret_cast<const ScoreT*>(&v);
#pragma unroll
                for (int i = 0; i < PER; ++i) s[i] = sv[i];
            }
            uint32_t gt = 0, eq = 0;
#pragma unroll
            for (int i = 0; i < PER; ++i) {
                const uint64_t row = my + i;
                const bool valid = row >= r0 && row < r1;
                gt += (valid && s[i] > T) ? 1u : 0u;
                eq += (valid && s[i] == T) ? 1u : 0u;
            }
            uint64_t tot;
            const uint64_t ex = block_excl_scan_u64(((uint64_t)eq << 32) | gt, s_warp, tot);
            if (gt | eq) {
                uint64_t eq_before = carry_eq + (ex >> 32);
                uint64_t pos = carry_gt + (ex & 0xffffffffu) + (eq_before < take ? eq_before : take);
#pragma unroll
                for (int i = 0; i < PER; ++i) {
                    const uint64_t row = my + i;
                    if (row < r0 || row >= r1) continue;
                    if (s[i] > T) {
                        out[pos++] = (uint32_t)row;
                    } else if (s[i] == T) {
                        if (eq_before < take) out[pos++] = (uint32_t)row;
                        ++eq_before;
                    }
                }
            }
            carry_gt += tot & 0xffffffffu;
            carry_eq += tot >> 32;
        }
    }
}

// Shard planning: one CTA per problem, from all ranks' histograms.
__global__ void __launch_bounds__(kThreads) k3_shard_plan(K3Params prm, const uint32_t* all_hist,
                                                          uint32_t R, uint32_t rank,
                                                          uint32_t* out_offset) {
    __shared__ uint64_t s_warp[kThreads / 32 + 1];
    __shared__ spl_shard_plan s_plan;
    const uint32_t p = blockIdx.x;
    const uint32_t L = prm.L;
    if (threadIdx.x == 0) {
        // O(R * L) integer arithmetic, identical to the host form.
        s_plan = spl_plan_shard(all_hist + (uint64_t)p * (L + 1), (uint64_t)prm.g.P * (L + 1), R,
                                rank, L, prm.k);
    }
    __syncthreads();
    const spl_shard_plan pl = s_plan;
    plan_segments(prm, p, pl.T, pl.take_eq, s_warp);
    if (threadIdx.x == 0) {
        prm.cnt_out[p] = pl.T == SPL_PLAN_SKIP ? 0u : pl.count;
        if (out_offset) out_offset[p] = pl.offset;
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
    if (zero) SPL_CUDA_TRY(ctx, cudaMemset(*buf, 0, want));
    *have = want;
    return SPL_OK;
}

namespace {

struct K3Plan {
    K3Geom g;
    bool vec;
    int hmode;
    size_t smem;
    size_t score_bytes;
};

size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

int hist_mode(uint32_t L) { return (size_t)(L + 1) * kThreads * 2 <= 150 * 1024 ? 0 : 1; }

size_t scan_smem(uint32_t L, int hmode) {
    if (hmode == 1) return (size_t)(L + 2) * 4;  // histogram reduced in place
    return align_up((size_t)(L + 1) * kThreads * 2, 16) + (size_t)(L + 2) * 4;
}

template <int W, typename ScoreT, int HM>
const void* scan_fn() {
    return reinterpret_cast<const void*>(&k3_scan<W, ScoreT, HM>);
}

template <typename ScoreT, int HM>
const void* pick_scan_w(uint32_t W) {
    switch (W) {
        case 1: return scan_fn<1, ScoreT, HM>();
        case 2: return scan_fn<2, ScoreT, HM>();
        case 4: return scan_fn<4, ScoreT, HM>();
        case 8: return scan_fn<8, ScoreT, HM>();
        default: return scan_fn<0, ScoreT, HM>();  // any W, 32-bit loads
    }
}

// vec: problem bases are 32-byte aligned (required by the 256-bit path).
const void* pick_scan(uint32_t L, int hmode, bool vec) {
    const uint32_t W = vec && (L / 32) <= 8 ? L / 32 : 0;
    if (L <= 255) return hmode == 0 ? pick_scan_w<uint8_t, 0>(W) : pick_scan_w<uint8_t, 1>(W);
    return hmode == 0 ? pick_scan_w<uint16_t, 0>(W) : pick_scan_w<uint16_t, 1>(W);
}

spl_status make_plan(spl_ctx* ctx, uint32_t P, uint64_t n_max, uint32_t L, const void* codes,
                     uint64_t stride_rows, K3Plan* out) {
    K3Plan pl{};
    const uint32_t W = L / 32;
    pl.vec = W <= 8 && 8 % W == 0 && (reinterpret_cast<uintptr_t>(codes) % 32) == 0 &&
             (stride_rows * W * 4) % 32 == 0;
    pl.hmode = hist_mode(L);
    pl.smem = scan_smem(L, pl.hmode);
    const void* fn = pick_scan(L, pl.hmode, pl.vec);
    SPL_CUDA_TRY(ctx, cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)pl.smem));
    int per_sm = 0;
    SPL_CUDA_TRY(ctx, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kThreads,
                                                                    pl.smem));
    if (per_sm < 1) per_sm = 1;
    const uint64_t total = (uint64_t)P * n_max;
    const uint64_t target = (uint64_t)ctx->num_sms * per_sm;
    uint64_t S = (total + target - 1) / target;
    S = align_up(std::max<uint64_t>(S, 1024), 256);
    S = std::min<uint64_t>(S, (uint64_t)65535 * kThreads);  // u16 private counters
    pl.g.n_max = n_max;
    pl.g.total = total;
    pl.g.S = S;
    pl.g.G = (uint32_t)((total + S - 1) / S);
    pl.g.P = P;
    pl.g.n_pad = align_up(n_max, 64);
    pl.score_bytes = L <= 255 ? 1 : 2;
    *out = pl;
    return SPL_OK;
}

struct K3Ws {
    void* scores;
    uint32_t* records;
    uint4* plans;
    uint32_t* counters;
    uint32_t* tot;
};

spl_status k3_workspace(spl_ctx* ctx, const K3Plan& pl, uint32_t L, cudaStream_t s, K3Ws* ws) {
    const size_t sc = align_up((size_t)pl.g.P * pl.g.n_pad * pl.score_bytes, 256);
    const size_t rec = align_up((size_t)(pl.g.G + pl.g.P) * (L + 2) * 4, 256);
    const size_t plans = align_up((size_t)(pl.g.G + pl.g.P) * 16, 256);
    spl_status st = ensure_buffer(ctx, &ctx->k3_ws, &ctx->k3_ws_bytes, sc + rec + plans, false, s,
                                  "hamming_topk");
    if (st) return st;
    const size_t state_words = (size_t)pl.g.P * (1 + (L + 2));
    size_t have = ctx->k3_state_words * 4;
    st = ensure_buffer(ctx, reinterpret_cast<void**>(&ctx->k3_state), &have, state_words * 4, true,
                       s, "hamming_topk");
    if (st) return st;
    ctx->k3_state_words = have / 4;
    uint8_t* b = static_cast<uint8_t*>(ctx->k3_ws);
    ws->scores = b;
    ws->records = reinterpret_cast<uint32_t*>(b + sc);
    ws->plans = reinterpret_cast<uint4*>(b + sc + rec);
    ws->counters = ctx->k3_state;
    ws->tot = ctx->k3_state + pl.g.P;
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
    const void* fn = pick_scan(prm.L, pl.hmode, pl.vec);
    void* args[] = {const_cast<K3Params*>(&prm)};
    SPL_CUDA_TRY(ctx, cudaLaunchKernel(fn, dim3(pl.g.G), dim3(kThreads), args, pl.smem, s));
    return after_launch(ctx, "k3_scan");
}

spl_status launch_select(spl_ctx* ctx, const K3Plan& pl, const K3Params& prm, uint32_t* idx,
                         uint64_t idx_stride, cudaStream_t s) {
    if (pl.score_bytes == 1)
        k3_select<uint8_t><<<pl.g.G, kThreads, 0, s>>>(prm, idx, idx_stride);
    else
        k3_select<uint16_t><<<pl.g.G, kThreads, 0, s>>>(prm, idx, idx_stride);
    return after_launch(ctx, "k3_select");
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
    if (n_max == 0 || n_max > 0xFFFFFFFFull) {
        if (n_max == 0) {
            SPL_CUDA_TRY(ctx, cudaMemsetAsync(cnt, 0, sizeof(uint32_t) * P, s));
            return SPL_OK;
        }
        return fail(ctx, SPL_E_DIMENSION, "hamming_topk: n_max exceeds 2^32 rows");
    }
    K3Plan pl;
    if ((st = make_plan(ctx, P, n_max, L, codes, stride_rows, &pl))) return st;
    K3Ws ws;
    if ((st = k3_workspace(ctx, pl, L, s, &ws))) return st;
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
    prm.tot_hist = ws.tot;
    prm.tot_stride = L + 2;
    prm.counters = ws.counters;
    prm.plans = ws.plans;
    prm.cnt_out = cnt;
    prm.dev_err = ctx->dev_err;
    prm.shard = 0;
    if ((st = launch_scan(ctx, pl, prm, s))) return st;
    return launch_select(ctx, pl, prm, idx, k, s);
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
    ctx->shard_G = pl.g.G;
    ctx->shard_S = pl.g.S;
    K3Params prm{};
    prm.codes = codes;
    prm.stride_rows = stride_rows;
    prm.qcodes = qcodes;
    prm.n_valid = n_valid;
    prm.nvalid_div = nvalid_div;
    prm.L = L;
    prm.W = L / 32;
    prm.k = 1;
    prm.g = pl.g;
    prm.scores = ws.scores;
    prm.records = ws.records;
    prm.tot_hist = hist;
    prm.tot_stride = L + 1;
    prm.counters = ws.counters;
    prm.plans = ws.plans;
    prm.cnt_out = nullptr;
    prm.dev_err = ctx->dev_err;
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
    pl.g.total = (uint64_t)P * n_max;
    pl.g.S = ctx->shard_S;
    pl.g.G = ctx->shard_G;
    pl.g.P = P;
    pl.g.n_pad = align_up(n_max, 64);
    pl.score_bytes = L <= 255 ? 1 : 2;
    K3Ws ws;
    if ((st = k3_workspace(ctx, pl, L, s, &ws))) return st;
    K3Params prm{};
    prm.n_valid = n_valid;
    prm.nvalid_div = nvalid_div;
    prm.L = L;
    prm.W = L / 32;
    prm.k = k;
    prm.g = pl.g;
    prm.scores = ws.scores;
    prm.records = ws.records;
    prm.plans = ws.plans;
    prm.cnt_out = cnt;
    prm.dev_err = ctx->dev_err;
    prm.shard = 1;
    k3_shard_plan<<<P, kThreads, 0, s>>>(prm, all_hist, R, rank, out_offset);
    if ((st = after_launch(ctx, "k3_shard_plan"))) return st;
    return launch_select(ctx, pl, prm, idx, k, s);
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
