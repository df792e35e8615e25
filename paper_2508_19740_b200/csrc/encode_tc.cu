// K2 — tcgen05 bulk key encoder (prefill / bulk re-encode), sm_100a.
//
// Same function as mlp_hash / linear_hash + pack_bits (hashers.cpp:75-82,
// :84-108; bitcodes.cpp:22-41) computed on the 5th-generation tensor cores in
// bf16 with fp32 accumulation — a fast mode: code bits can differ from the
// exact encoder (K1, bit-identical with the reference) only where a
// pre-activation lies within the bf16 rounding band around 0.
//
// One CTA (256 threads) per SM walks a contiguous range of 128-key tiles
// (tiles of one (b, head) problem are consecutive, so the head's weights are
// reloaded only when the range crosses a problem boundary):
//   X tile [128 x 128] f32/bf16 -> bf16, swizzled (spl_tc.cuh) into smem
//   GEMM1  D1[128 x 128] = X . W1          tcgen05.mma kind::f16, TMEM cols [0,128)
//   epi 1  +b1, SiLU (fp32) -> bf16 A1 in smem (8 warps: lane quarter x column half)
//   GEMM2  D2[128 x L] = A1 . W2           TMEM cols [128, 128+L)
//   epi 2  bit = (z2 >= 0) -> Appendix A.7 words (column j -> word j % W,
//          bit 31 - j / W), column halves OR-ed through smem, one store per row
// linear_hash: GEMM1 with N = L and epilogue 2 straight from D1.
// One thread issues the MMAs (8 k-steps of 16); tcgen05.commit -> mbarrier
// tells the epilogue warps the accumulator is ready. The next tile's X is
// staged while GEMM2 and epilogue 2 of the current tile run (sX is free once
// GEMM1 has committed).
//
// Roofline (SURVEY §8 d, config 4 prefill): 98,304 FLOP per key (2dh + 2hL,
// d = h = L = 128: 65,536; L = 256: 98,304) against 256 B (bf16) or 512 B
// (f32) of input per key: bf16 input at L = 256 is at/above the ridge.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "spl_launch.cuh"
#include "spl_tc.cuh"

namespace spl {
namespace {

constexpr int kTcThreads = 256;

struct TcParams {
    const void* x;  // [B][H][m][128] f32 or bf16
    int x_bf16;
    uint32_t H, m, L, W;
    int linear;
    const uint8_t* w1_tc;  // [H][N1 x 256 B] swizzled bf16 (N1 = 128, linear: L)
    const uint8_t* w2_tc;  // [H][L x 256 B]
    const float* b1;       // [H][128]
    uint32_t* codes;       // [B][H][m][W]
    float* pre;            // optional [B][H][m][L] pre-activations (tests)
    uint32_t tiles_per_problem;
    uint64_t total_tiles;
    uint32_t* dev_err;
    long long* trace;  // optional (SPL_K2_TRACE=<first tile>): CTA 0's per-tile role clocks [64][12]
    uint32_t trace_from;
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}

// shared-memory matrix descriptor: K-major, SWIZZLE_128B, SBO = 1024 B
// (8-row atoms), LBO = 16 B (unused for swizzled K-major), version 1 (sm_100)
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr) {
    return (uint64_t)((saddr >> 4) & 0x3FFFu) | (1ull << 16) | ((uint64_t)(1024u >> 4) << 32) |
           (1ull << 46) | (2ull << 61);
}
// instruction descriptor, kind::f16: D f32, A/B bf16, both K-major, M = 128
__device__ __forceinline__ uint32_t umma_idesc(uint32_t N) {
    return (1u << 4) | (1u << 7) | (1u << 10) | ((N >> 3) << 17) | ((kTcTileM >> 4) << 24);
}
__device__ __forceinline__ void umma_bf16(uint32_t tmem_d, uint64_t da, uint64_t db,
                                          uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
        "l"(da), "l"(db), "r"(idesc), "r"(acc));
}
// D[128 x N] = A[128 x 128] . B[N x 128]^T (operands as in spl_tc.cuh)
__device__ __forceinline__ void gemm_k128(uint32_t tmem_d, uint32_t sa, uint32_t sb, uint32_t N) {
    const uint32_t idesc = umma_idesc(N);
#pragma unroll
    for (uint32_t s = 0; s < kTcK / 16; ++s) {
        const uint64_t da = umma_desc(sa + (s >> 2) * kTcTileM * 128u + (s & 3u) * 32u);
        const uint64_t db = umma_desc(sb + (s >> 2) * N * 128u + (s & 3u) * 32u);
        umma_bf16(tmem_d, da, db, idesc, s > 0 ? 1u : 0u);
    }
}
// D[128 x N] = A[128 x 128] . B[N x 128]^T with A in TMEM (row r = lane r,
// k-step s = 16 bf16 = columns [8s, 8s + 8), element 2c in the low half of
// column c) and B in shared memory as in gemm_k128
__device__ __forceinline__ void gemm_k128_ta(uint32_t tmem_d, uint32_t tmem_a, uint32_t sb, uint32_t N) {
    const uint32_t idesc = umma_idesc(N);
#pragma unroll
    for (uint32_t s = 0; s < kTcK / 16; ++s) {
        const uint64_t db = umma_desc(sb + (s >> 2) * N * 128u + (s & 3u) * 32u);
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(tmem_d),
            "r"(tmem_a + 8u * s), "l"(db), "r"(idesc), "r"(s > 0 ? 1u : 0u));
    }
}
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&r)[32]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
        "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
        "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]),
        "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]),
        "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
        : "memory");
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                     smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    uint32_t done = 0;
    while (!done)
        asm volatile(
            "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
            : "=r"(done)
            : "r"(smem_u32(bar)), "r"(parity)
            : "memory");
}
// Same with a suspend-time hint: the waiting warp sleeps until the phase
// completes (or ~hint ns pass) instead of re-issuing try_wait. In the
// warp-specialised kernel the spinning of the MMA / producer / epilogue
// waits was ~20 % of all issued instructions, taking issue slots from the
// epilogue warps on the same SMSP.
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, uint32_t parity) {
    uint32_t done = 0;
    while (!done)
        asm volatile(
            "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3; selp.u32 %0, 1, 0, p; }"
            : "=r"(done)
            : "r"(smem_u32(bar)), "r"(parity), "r"(1000000u)
            : "memory");
}
__device__ __forceinline__ void fence_before() {
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void fence_after() {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
// generic-proxy smem writes -> visible to the tensor core (async proxy)
__device__ __forceinline__ void fence_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {
    const __nv_bfloat162 t = __floats2bfloat162_rn(a, b);
    return *reinterpret_cast<const uint32_t*>(&t);
}

// Stage X rows [row0, row0 + 128) of problem bh into sX (bf16, swizzled);
// rows >= m are zero. Non-finite input raises the device error word.
__device__ __forceinline__ void stage_x(const TcParams& prm, uint64_t bh, uint32_t row0, uint8_t* sX) {
    const int tid = threadIdx.x;
    bool bad = false;
#pragma unroll 2
    for (uint32_t it = tid; it < kTcTileM * 16; it += kTcThreads) {
        const uint32_t r = it >> 4, c = it & 15u, gr = row0 + r;
        uint4 v = make_uint4(0, 0, 0, 0);
        if (gr < prm.m) {
            const uint64_t e = ((bh * prm.m) + gr) * kTcK + c * 8;
            if (prm.x_bf16) {
                v = __ldg(reinterpret_cast<const uint4*>(static_cast<const __nv_bfloat16*>(prm.x) + e));
                const __nv_bfloat16* h = reinterpret_cast<const __nv_bfloat16*>(&v);
#pragma unroll
                for (int i = 0; i < 8; ++i) bad |= !isfinite(__bfloat162float(h[i]));
            } else {
                const float4* p = reinterpret_cast<const float4*>(static_cast<const float*>(prm.x) + e);
                const float4 a = __ldg(p), b = __ldg(p + 1);
                bad |= !(isfinite(a.x) && isfinite(a.y) && isfinite(a.z) && isfinite(a.w) &&
                         isfinite(b.x) && isfinite(b.y) && isfinite(b.z) && isfinite(b.w));
                v = make_uint4(pack_bf16(a.x, a.y), pack_bf16(a.z, a.w), pack_bf16(b.x, b.y),
                               pack_bf16(b.z, b.w));
            }
        }
        *reinterpret_cast<uint4*>(sX + tc_sw_off(r, c * 8, kTcTileM)) = v;
    }
    if (bad) raise_dev_err(prm.dev_err, SPL_DEV_ERR_NUMERIC);
}

// SiLU with one MUFU op: z * sigmoid(z) = h (1 + tanh h), h = z / 2, as
// fma(h, tanh h, h) (the warp-specialised kernel computes the same h as
// fma(acc, 1/2, b1/2), so both kernels round identically)
__device__ __forceinline__ float silu_fast(float z) {
    const float h = 0.5f * z;
    float t;
    asm("tanh.approx.f32 %0, %1;" : "=f"(t) : "f"(h));
    return fmaf(h, t, h);
}

__device__ __forceinline__ void tma_x(const CUtensorMap* tmap, uint8_t* dst, uint64_t* bar,
                                      uint64_t row) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(tc_operand_bytes(kTcTileM))
                 : "memory");
#pragma unroll
    for (uint32_t kb = 0; kb < 2; ++kb)
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::
                "r"(smem_u32(dst + kb * kTcTileM * 128u)),
            "l"(reinterpret_cast<uint64_t>(tmap)), "r"(kb * 64u), "r"((uint32_t)row), "r"(smem_u32(bar))
            : "memory");
}

__device__ __forceinline__ void tmem_ld16_nowait(uint32_t taddr, uint32_t (&r)[16]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
          "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
          "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
}
__device__ __forceinline__ void tmem_ld32_nowait(uint32_t taddr, uint32_t (&r)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
          "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
          "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]),
          "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]),
          "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// Epilogue 2 for one column half: code bit of column j = (z_j >= 0) goes to
// word j % W, bit 31 - j / W (Appendix A.7). Collects NEGATIVE flags (raw
// sign bits) with compile-time shifts; the word is the complement. A z2 of
// exactly -0.0 (every product of its dot a signed zero) gets bit 0 where the
// exact encoder gives 1: K2 is the fast mode, whose bits may differ from the
// exact ones only inside the rounding band around 0, and -0.0 is at 0. `sum` accumulates the values
// (non-finite check). Two TMEM loads in flight per wait.
template <uint32_t W, uint32_t HALF>
__device__ __forceinline__ void sign_half(uint32_t tz, uint32_t (&neg)[W], float& sum) {
    constexpr uint32_t L = 32 * W, NCH = W;  // W chunks of 16 columns per half
#pragma unroll
    for (uint32_t cp = 0; cp < NCH; cp += 2) {
        uint32_t r[2][16];
        tmem_ld16_nowait(tz + HALF * (L / 2) + 16 * cp, r[0]);
        if (cp + 1 < NCH) tmem_ld16_nowait(tz + HALF * (L / 2) + 16 * (cp + 1), r[1]);
        tmem_wait_ld();
#pragma unroll
        for (uint32_t q = 0; q < 2; ++q) {
            if (cp + q >= NCH) break;
            const uint32_t c0 = HALF * (L / 2) + 16 * (cp + q);
#pragma unroll
            for (uint32_t i = 0; i < 16; ++i) {
                const float z = __uint_as_float(r[q][i]);
                sum += z;
                const uint32_t u = r[q][i];
                const uint32_t sh = (c0 + i) / W;
                neg[(c0 + i) % W] |= (u >> sh) & (0x80000000u >> sh);
            }
        }
    }
}

// TMA_X: bf16 input through a 2-D tensor map (128-byte swizzle = the UMMA
// operand layout) into a 2-slot ring, issued two tiles ahead; otherwise (f32
// input) all threads convert and stage the tile two ahead once its slot is free.
template <bool TMA_X, uint32_t W>
__global__ void __launch_bounds__(kTcThreads, 1)
    k2_encode_tc(const __grid_constant__ CUtensorMap tmap, TcParams prm) {
    extern __shared__ uint8_t smem_raw[];
    __shared__ __align__(8) uint64_t s_bar[4];  // [0,1] X slot full, [2] GEMM1 done, [3] GEMM2 done
    __shared__ uint32_t s_tmem;
    __shared__ float s_b1[kTcK];
    constexpr uint32_t L = 32 * W;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t N1 = prm.linear ? L : kTcK;
    const uint32_t base_s = (smem_u32(smem_raw) + 1023u) & ~1023u;
    uint8_t* base = smem_raw + (base_s - smem_u32(smem_raw));
    uint8_t* sX0 = base;  // 2 slots
    uint8_t* sA1 = sX0 + 2 * tc_operand_bytes(kTcTileM);
    uint8_t* sW1 = sA1 + tc_operand_bytes(kTcTileM);
    uint8_t* sW2 = sW1 + tc_operand_bytes(N1);
    uint32_t* s_code = reinterpret_cast<uint32_t*>(sW2 + (prm.linear ? 0u : tc_operand_bytes(L)));
    auto sX = [&](uint64_t t) { return sX0 + (t & 1) * tc_operand_bytes(kTcTileM); };

    const uint64_t T = prm.total_tiles;
    const uint32_t tpp = prm.tiles_per_problem;
    const uint64_t t0 = T * blockIdx.x / gridDim.x, t1 = T * (blockIdx.x + 1) / gridDim.x;
    // tile t <-> (problem bh, tile-in-problem mb), head = bh % H; walked incrementally
    struct Pos {
        uint64_t bh;
        uint32_t mb, head;
    };
    auto pos_of = [&](uint64_t t) {
        Pos p;
        p.bh = t / tpp;
        p.mb = (uint32_t)(t - p.bh * tpp);
        p.head = (uint32_t)(p.bh % prm.H);
        return p;
    };
    auto next = [&](Pos p) {
        if (++p.mb == tpp) {
            p.mb = 0;
            ++p.bh;
            if (++p.head == prm.H) p.head = 0;
        }
        return p;
    };
    auto stage = [&](uint64_t t, Pos p) {  // bring tile t's keys into its slot
        if (TMA_X) {
            if (tid == 0) tma_x(&tmap, sX(t), &s_bar[t & 1], p.bh * prm.m + (uint64_t)p.mb * kTcTileM);
        } else {
            stage_x(prm, p.bh, p.mb * kTcTileM, sX(t));
        }
    };
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                         smem_u32(&s_tmem))
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    if (tid == 0) {
        for (int i = 0; i < 4; ++i)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&s_bar[i])));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        if (TMA_X) asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmap)) : "memory");
    }
    fence_before();
    __syncthreads();
    fence_after();
    const uint32_t tmem = s_tmem;
    const uint32_t tD1 = tmem, tD2 = tmem + kTcK;
    const uint32_t quarter = (uint32_t)(warp & 3), half = (uint32_t)(warp >> 2);
    const uint32_t row = quarter * 32 + lane;  // this thread's TMEM lane = tile row
    const uint32_t lane_addr = (quarter * 32) << 16;

    uint32_t xph = 0, g1ph = 0, g2ph = 0;  // xph bit s: parity of X slot s
    uint32_t cur_head = ~0u;
    bool g1_issued = false;  // GEMM1 of the current tile already in flight
    Pos pc = pos_of(t0 < t1 ? t0 : 0);
    if (t0 < t1) stage(t0, pc);
    Pos pn = next(pc), pnn = next(pn);
    if (t0 + 1 < t1) stage(t0 + 1, pn);
    auto load_weights = [&](uint32_t head) {
        const uint4* g1 = reinterpret_cast<const uint4*>(prm.w1_tc + (uint64_t)head * tc_operand_bytes(N1));
        for (uint32_t i = tid; i < tc_operand_bytes(N1) / 16; i += kTcThreads)
            reinterpret_cast<uint4*>(sW1)[i] = __ldg(g1 + i);
        if (!prm.linear) {
            const uint4* g2 = reinterpret_cast<const uint4*>(prm.w2_tc + (uint64_t)head * tc_operand_bytes(L));
            for (uint32_t i = tid; i < tc_operand_bytes(L) / 16; i += kTcThreads)
                reinterpret_cast<uint4*>(sW2)[i] = __ldg(g2 + i);
            for (uint32_t i = tid; i < kTcK; i += kTcThreads) s_b1[i] = prm.b1[(uint64_t)head * kTcK + i];
        }
    };
    auto issue_g1 = [&](uint64_t t) {  // thread 0 only
        if (TMA_X) mbar_wait(&s_bar[t & 1], (xph >> (t & 1)) & 1u);
        fence_after();
        gemm_k128(tD1, smem_u32(sX(t)), smem_u32(sW1), N1);
        umma_commit(&s_bar[2]);
    };
    for (uint64_t t = t0; t < t1; ++t) {
        if (!g1_issued) {
            if (pc.head != cur_head) {  // all earlier MMAs are complete here
                load_weights(pc.head);
                cur_head = pc.head;
            }
            fence_async_smem();
            fence_before();
            __syncthreads();
            if (tid == 0) issue_g1(t);
        }
        xph ^= 1u << (t & 1);
        // ---- GEMM1(t) done: its X slot is free for tile t + 2
        mbar_wait(&s_bar[2], g1ph);
        g1ph ^= 1u;
        fence_after();
        if (t + 2 < t1) stage(t + 2, pnn);
        uint32_t tZ = tD1;
        // GEMM1(t + 1) runs under epilogue 2 of tile t when its weights (head)
        // are already loaded and D1 is not the final accumulator (MLP)
        const bool early = !prm.linear && t + 1 < t1 && pn.head == pc.head;
        if (!prm.linear) {
            // ---- epilogue 1: +b1, SiLU -> bf16 A1 (columns [64 half, +64))
#pragma unroll
            for (uint32_t cc = 0; cc < 64; cc += 32) {
                const uint32_t c0 = half * 64 + cc;
                uint32_t r[2][16];
                tmem_ld16_nowait(tD1 + lane_addr + c0, r[0]);
                tmem_ld16_nowait(tD1 + lane_addr + c0 + 16, r[1]);
                tmem_wait_ld();
#pragma unroll
                for (uint32_t q = 0; q < 2; ++q) {
                    uint32_t p[8];
#pragma unroll
                    for (int i = 0; i < 16; i += 2)
                        p[i / 2] = pack_bf16(silu_fast(__uint_as_float(r[q][i]) + s_b1[c0 + 16 * q + i]),
                                             silu_fast(__uint_as_float(r[q][i + 1]) + s_b1[c0 + 16 * q + i + 1]));
                    *reinterpret_cast<uint4*>(sA1 + tc_sw_off(row, c0 + 16 * q, kTcTileM)) =
                        make_uint4(p[0], p[1], p[2], p[3]);
                    *reinterpret_cast<uint4*>(sA1 + tc_sw_off(row, c0 + 16 * q + 8, kTcTileM)) =
                        make_uint4(p[4], p[5], p[6], p[7]);
                }
            }
            fence_async_smem();
            fence_before();
            __syncthreads();
            // ---- GEMM2(t), then GEMM1(t + 1) (D1 has been drained)
            if (tid == 0) {
                fence_after();
                gemm_k128(tD2, smem_u32(sA1), smem_u32(sW2), L);
                umma_commit(&s_bar[3]);
                if (early) issue_g1(t + 1);
            }
            tZ = tD2;
            mbar_wait(&s_bar[3], g2ph);
            g2ph ^= 1u;
            fence_after();
        }
        g1_issued = early;
        // ---- epilogue 2: this half's columns -> negative flags -> code words
        uint32_t neg[W];
#pragma unroll
        for (uint32_t w = 0; w < W; ++w) neg[w] = 0u;
        float sum = 0.0f;
        if (half == 0) sign_half<W, 0>(tZ + lane_addr, neg, sum);
        else sign_half<W, 1>(tZ + lane_addr, neg, sum);
        const uint32_t grow = pc.mb * kTcTileM + row;
        if (TMA_X && !isfinite(sum) && grow < prm.m) raise_dev_err(prm.dev_err, SPL_DEV_ERR_NUMERIC);
        if (prm.pre) {  // tests: the f32 pre-activations of this half (tcgen05.ld
                        // is warp-collective: load on every lane, store if valid)
            float* dst = prm.pre + ((pc.bh * prm.m) + grow) * L + half * (L / 2);
            for (uint32_t c = 0; c < L / 2; c += 16) {
                uint32_t r[16];
                tmem_ld16_nowait(tZ + lane_addr + half * (L / 2) + c, r);
                tmem_wait_ld();
                if (grow < prm.m)
                    for (int i = 0; i < 16; ++i) dst[c + i] = __uint_as_float(r[i]);
            }
        }
        if (half == 1) {
#pragma unroll
            for (uint32_t w = 0; w < W; ++w) s_code[row * 8 + w] = neg[w];
        }
        fence_before();
        __syncthreads();
        if (half == 0 && grow < prm.m) {
            uint32_t wd[W];
#pragma unroll
            for (uint32_t w = 0; w < W; ++w) wd[w] = ~(neg[w] | s_code[row * 8 + w]);
            uint32_t* dst = prm.codes + ((pc.bh * prm.m) + grow) * W;
            if constexpr (W >= 4) {
#pragma unroll
                for (uint32_t w = 0; w < W; w += 4)
                    *reinterpret_cast<uint4*>(dst + w) = make_uint4(wd[w], wd[w + 1], wd[w + 2], wd[w + 3]);
            } else {
#pragma unroll
                for (uint32_t w = 0; w < W; ++w) dst[w] = wd[w];
            }
        }
        pc = pn;
        pn = pnn;
        pnn = next(pnn);
    }
    fence_before();
    __syncthreads();
    fence_after();
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
}

// ---------------------------------------------------------------------------
// Warp-specialised MLP encoder (bf16 keys via TMA, no pre-activation dump):
// the production prefill path. The single-CTA-team kernel above runs GEMM1 ->
// epilogue 1 -> GEMM2 -> epilogue 2 as one chain per tile, so the tensor pipe
// idles while the CUDA cores work (~42% of peak). Here every stage has its
// own warps and its own buffers, handshaking through mbarriers, so GEMM1 of
// tile i+1 and GEMM2 of tile i-1 run under epilogue 1 of tile i and
// epilogue 2 of tile i-1:
//   warp 0 (lane 0)  MMA issuer: GEMM1(i) -> D1[i&1], GEMM2(i-1) -> D2
//   warp 1 (lane 0)  producer: X tiles (TMA, 2 slots), per-head W1/W2 (bulk copy)
//   warps 2-9        epilogue 1: D1 -> +b1, SiLU -> bf16 A1[i&1] (smem); two
//                    warps per lane quarter (column halves): it is the
//                    busiest stage (MUFU tanh + packing), one warp per SMSP
//                    could not hide its latencies
//   warps 10-13      epilogue 2: D2 -> sign bits -> Appendix A.7 code words
// TMEM: D1[0] cols [0,128), D1[1] [128,256), D2 [256, 256+L) (512 allocated).
// Shared: X 2 x 32 KB, A1 2 x 32 KB, W1 32 KB, W2 L x 256 B (<= 224 KB).
// A warp may only touch the TMEM lane quarter warp % 4, so each epilogue
// group is 4 consecutive warps covering the 4 quarters; thread = tile row.
constexpr int kWsThreads = 448;
constexpr uint32_t kEpi1Threads = 256;
// tile t <-> (problem bh, tile-in-problem mb, head = bh % H), advanced one
// tile at a time (a 64-bit divide per tile per role cost ~17% of the samples)
struct TilePos {
    uint64_t bh;
    uint32_t mb, head, tpp, H;
    __device__ TilePos(uint64_t t, uint32_t tpp_, uint32_t H_) : tpp(tpp_), H(H_) {
        bh = t / tpp;
        mb = (uint32_t)(t - bh * tpp);
        head = (uint32_t)(bh % H);
    }
    __device__ __forceinline__ void advance() {
        if (++mb == tpp) {
            mb = 0;
            ++bh;
            if (++head == H) head = 0;
        }
    }
    __device__ __forceinline__ bool last_of_head() const { return mb + 1 == tpp; }
};
constexpr uint32_t kXSlots = 4;  // X ring depth (A1 lives in TMEM: its 64 KB went to X)
enum WsBar {
    kXFull = 0,      // [4] producer -> MMA (TMA tx)
    kXEmpty = 4,     // [4] GEMM1 done reading X
    kD1Full = 8,     // [2] GEMM1 done -> epilogue 1
    kA1Full = 10,    // [2] epilogue 1 wrote A1 into the D1 slot (256 arrivals)
    kD2Full = 12,    // GEMM2 done -> epilogue 2
    kD2Empty = 13,   // epilogue 2 drained D2 (128 arrivals)
    kWFull = 14,     // head weights landed (bulk tx)
    kWEmpty = 15,    // last GEMM2 of a head done: weights may be replaced
    kWsBars = 16
};

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

#define K2T(i, k)                                                                      \
    if (prm.trace && blockIdx.x == 0 && (i) >= prm.trace_from && (i) < prm.trace_from + 64 && \
        (threadIdx.x & 31) == 0)                                                           \
    prm.trace[((i) - prm.trace_from) * 12 + (k)] = clock64()

template <uint32_t W>
__global__ void __launch_bounds__(kWsThreads, 1)
    k2_encode_ws(const __grid_constant__ CUtensorMap tmap, TcParams prm) {
    extern __shared__ uint8_t smem_raw[];
    __shared__ __align__(8) uint64_t bar[kWsBars];
    __shared__ uint32_t s_tmem;
    __shared__ __align__(16) float s_b1[kTcK];  // epilogue 1's bias of the current head
    constexpr uint32_t L = 32 * W;
    constexpr uint32_t XB = kTcTileM * 256u;  // one 128 x 128 bf16 operand
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t base_s = (smem_u32(smem_raw) + 1023u) & ~1023u;
    uint8_t* base = smem_raw + (base_s - smem_u32(smem_raw));
    uint8_t* sX = base;             // kXSlots slots
    uint8_t* sW1 = sX + kXSlots * XB;
    uint8_t* sW2 = sW1 + XB;

    const uint64_t T = prm.total_tiles;
    const uint32_t tpp = prm.tiles_per_problem;
    const uint64_t t0 = T * blockIdx.x / gridDim.x, t1 = T * (blockIdx.x + 1) / gridDim.x;
    const uint32_t n = (uint32_t)(t1 - t0);

    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                         smem_u32(&s_tmem))
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    if (tid == 32) {
        for (int i = 0; i < kWsBars; ++i) {
            const bool e1 = i >= kA1Full && i < kA1Full + 2;
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&bar[i])),
                         "r"(e1 ? kEpi1Threads : i == kD2Empty ? 128u : 1u));
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmap)) : "memory");
    }
    fence_before();
    __syncthreads();
    fence_after();
    const uint32_t tmem = s_tmem;

    if (warp == 0) {
        // ------------------------------------------------ MMA issuer
        if (lane == 0 && n > 0) {
            uint32_t nw = 0;
            // a head's weights are last used by GEMM2 of a tile that ends its
            // problem (consecutive problems have consecutive heads; H = 1
            // reloads the same head, harmless)
            auto g2 = [&](uint32_t j, bool ends_head) {
                K2T(j, 2);
                mbar_wait(&bar[kA1Full + (j & 1)], (j >> 1) & 1u);
                K2T(j, 3);
                if (j >= 1) mbar_wait(&bar[kD2Empty], (j - 1) & 1u);
                fence_after();
                K2T(j, 4);
                // A1(j) in TMEM, in the D1 slot it was computed from; GEMM1(j + 2)
                // reuses the slot only after this GEMM2 (tcgen05.mma runs in issue order)
                gemm_k128_ta(tmem + 256u, tmem + (j & 1) * 128u, smem_u32(sW2), L);
                umma_commit(&bar[kD2Full]);
                if (j + 1 < n && ends_head) umma_commit(&bar[kWEmpty]);
            };
            TilePos pos(t0, tpp, prm.H);
            bool prev_ends = false;
            for (uint32_t i = 0; i < n; ++i) {
                const bool newhead = i == 0 || prev_ends;
                if (newhead) {
                    // the previous head's last GEMM2 goes first: the producer
                    // may only replace W1/W2 once it has completed
                    if (i >= 1) g2(i - 1, true);
                    mbar_wait(&bar[kWFull], nw & 1u);
                    ++nw;
                }
                K2T(i, 0);
                const uint32_t xs = i % kXSlots;
                mbar_wait(&bar[kXFull + xs], (i / kXSlots) & 1u);
                fence_after();
                K2T(i, 1);
                gemm_k128(tmem + (i & 1) * 128u, smem_u32(sX + xs * XB), smem_u32(sW1), kTcK);
                umma_commit(&bar[kXEmpty + xs]);
                umma_commit(&bar[kD1Full + (i & 1)]);
                if (i >= 1 && !newhead) g2(i - 1, false);
                prev_ends = pos.last_of_head();
                pos.advance();
            }
            g2(n - 1, false);
        }
    } else if (warp == 1) {
        // ------------------------------------------------ producer
        if (lane == 0) {
            uint32_t nw = 0;
            TilePos pos(t0, tpp, prm.H);
            bool prev_ends = false;
            for (uint32_t i = 0; i < n; ++i) {
                const uint32_t h = pos.head;
                if (i == 0 || prev_ends) {
                    if (nw > 0) mbar_wait_sleep(&bar[kWEmpty], (nw - 1) & 1u);
                    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(
                                     smem_u32(&bar[kWFull])),
                                 "r"(XB + L * 256u)
                                 : "memory");
                    bulk_g2s(sW1, prm.w1_tc + (uint64_t)h * XB, XB, &bar[kWFull]);
                    bulk_g2s(sW2, prm.w2_tc + (uint64_t)h * L * 256u, L * 256u, &bar[kWFull]);
                    ++nw;
                }
                K2T(i, 8);
                const uint32_t xs = i % kXSlots;
                if (i >= kXSlots) mbar_wait_sleep(&bar[kXEmpty + xs], ((i - kXSlots) / kXSlots) & 1u);
                K2T(i, 9);
                tma_x(&tmap, sX + xs * XB, &bar[kXFull + xs], pos.bh * prm.m + (uint64_t)pos.mb * kTcTileM);

                prev_ends = pos.last_of_head();
                pos.advance();
            }
        }
    } else if (warp < 10) {
        // ------------------------------------------------ epilogue 1
        const uint32_t q = (uint32_t)(warp & 3);
        const uint32_t ch = (uint32_t)(warp - 2) >> 2;  // column half
        const uint32_t lane_addr = (q * 32) << 16;
        const int et = tid - 64;  // 0..255 within the group
        TilePos pos(t0, tpp, prm.H);
        uint32_t cur_head = ~0u;
        for (uint32_t i = 0; i < n; ++i, pos.advance()) {
            if (pos.head != cur_head) {  // the group's own copy of b1 / 2 (named barrier 1)
                asm volatile("bar.sync 1, 256;" ::: "memory");
                if (et < (int)kTcK) s_b1[et] = 0.5f * __ldg(prm.b1 + (uint64_t)pos.head * kTcK + et);
                asm volatile("bar.sync 1, 256;" ::: "memory");
                cur_head = pos.head;
            }
            mbar_wait_sleep(&bar[kD1Full + (i & 1)], (i >> 1) & 1u);
            fence_after();
            if (warp == 2) K2T(i, 5);
            // this thread's half row of D1 (64 columns) -> SiLU -> bf16 pairs
            // -> A1 columns [32 ch, 32 ch + 32) of the same TMEM slot (k-major
            // A operand of GEMM2: unit j at column j / 2, half j % 2)
            const uint32_t tS = tmem + (i & 1) * 128u + lane_addr;
            const uint32_t tD = tS + ch * 64u;
            uint32_t rr[2][32];
            tmem_ld32_nowait(tD, rr[0]);
            tmem_ld32_nowait(tD + 32, rr[1]);
            tmem_wait_ld();
            // both column halves of the quarter have their D1 values in
            // registers before either overwrites part of D1 with A1
            fence_before();
            asm volatile("bar.sync 1, 256;" ::: "memory");
            fence_after();
            uint32_t pk[32];
#pragma unroll
            for (uint32_t c0 = 0; c0 < 64; c0 += 32) {
                uint32_t (&r)[32] = rr[c0 >> 5];
#pragma unroll
                for (uint32_t hh = 0; hh < 2; ++hh) {
                    const float4* bp = reinterpret_cast<const float4*>(s_b1 + ch * 64u + c0 + 16 * hh);
                    float hb[16];  // b1 / 2
#pragma unroll
                    for (int v = 0; v < 4; ++v) {
                        const float4 x = bp[v];
                        hb[4 * v] = x.x; hb[4 * v + 1] = x.y; hb[4 * v + 2] = x.z; hb[4 * v + 3] = x.w;
                    }
#pragma unroll
                    for (int e = 0; e < 16; e += 2) {
                        // SiLU(z) = h (1 + tanh h), h = z / 2 = acc / 2 + b1 / 2
                        float a[2];
#pragma unroll
                        for (int u = 0; u < 2; ++u) {
                            const float hv = fmaf(__uint_as_float(r[16 * hh + e + u]), 0.5f, hb[e + u]);
                            float t;
                            asm("tanh.approx.f32 %0, %1;" : "=f"(t) : "f"(hv));
                            a[u] = fmaf(hv, t, hv);
                        }
                        pk[(c0 + 16 * hh + e) / 2] = pack_bf16(a[0], a[1]);
                    }
                }
            }
            tmem_st32(tS + ch * 32u, pk);
            asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
            fence_before();
            mbar_arrive(&bar[kA1Full + (i & 1)]);
            if (warp == 2) K2T(i, 6);
        }
    } else {
        // ------------------------------------------------ epilogue 2
        const uint32_t q = (uint32_t)(warp & 3), row = q * 32 + lane;
        const uint32_t tD = tmem + 256u + ((q * 32) << 16);
        TilePos pos(t0, tpp, prm.H);
        for (uint32_t i = 0; i < n; ++i, pos.advance()) {
            const uint64_t bh = pos.bh;
            const uint32_t grow = pos.mb * kTcTileM + row;
            mbar_wait_sleep(&bar[kD2Full], i & 1u);
            fence_after();
            if (warp == 10) K2T(i, 7);
            // column j -> word j % W, bit 31 - j / W: feeding the sign bits of
            // columns w, w + W, w + 2W, ... into word w with a funnel shift
            // puts column w + W*b at bit 31 - b. Raw sign bits (see sign_half
            // for -0.0): one funnel shift per column.
            uint32_t neg[W];
#pragma unroll
            for (uint32_t w = 0; w < W; ++w) neg[w] = 0u;
            // non-finite input: any NaN / Inf in a key row reaches every z1
            // column (x * w, NaN * 0 = NaN), every a1 and every z2 column, so
            // column 0 of D2 decides the row (one check instead of L)
            float z0 = 0.0f;
            constexpr uint32_t kCols = L >= 64 ? 64u : 32u;  // columns per TMEM wait
#pragma unroll
            for (uint32_t c0 = 0; c0 < L; c0 += kCols) {
                uint32_t r[kCols / 32][32];
#pragma unroll
                for (uint32_t h = 0; h < kCols / 32; ++h) tmem_ld32_nowait(tD + c0 + 32 * h, r[h]);
                tmem_wait_ld();
#pragma unroll
                for (uint32_t e = 0; e < kCols; ++e) {
                    const uint32_t u = r[e >> 5][e & 31];
                    if (c0 == 0 && e == 0) z0 = __uint_as_float(u);
                    neg[(c0 + e) % W] = __funnelshift_l(u, neg[(c0 + e) % W], 1);
                }
            }
            fence_before();
            mbar_arrive(&bar[kD2Empty]);
            if (grow < prm.m) {
                if (!isfinite(z0)) raise_dev_err(prm.dev_err, SPL_DEV_ERR_NUMERIC);
                uint32_t* dst = prm.codes + ((bh * prm.m) + grow) * W;
                if constexpr (W >= 4) {
#pragma unroll
                    for (uint32_t w = 0; w < W; w += 4)
                        *reinterpret_cast<uint4*>(dst + w) =
                            make_uint4(~neg[w], ~neg[w + 1], ~neg[w + 2], ~neg[w + 3]);
                } else {
#pragma unroll
                    for (uint32_t w = 0; w < W; ++w) dst[w] = ~neg[w];
                }
            }
        }
    }
    fence_before();
    __syncthreads();
    fence_after();
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
}

const void* k2_ws_fn(uint32_t W) {
    switch (W) {
        case 1: return reinterpret_cast<const void*>(&k2_encode_ws<1>);
        case 2: return reinterpret_cast<const void*>(&k2_encode_ws<2>);
        case 4: return reinterpret_cast<const void*>(&k2_encode_ws<4>);
        default: return reinterpret_cast<const void*>(&k2_encode_ws<8>);
    }
}

template <bool TMA_X>
const void* k2_fn(uint32_t W) {
    switch (W) {
        case 1: return reinterpret_cast<const void*>(&k2_encode_tc<TMA_X, 1>);
        case 2: return reinterpret_cast<const void*>(&k2_encode_tc<TMA_X, 2>);
        case 4: return reinterpret_cast<const void*>(&k2_encode_tc<TMA_X, 4>);
        default: return reinterpret_cast<const void*>(&k2_encode_tc<TMA_X, 8>);
    }
}

}  // namespace

bool encode_tc_eligible(uint32_t kind, uint32_t d, uint32_t h, uint32_t L) {
    const bool l_ok = L == 32 || L == 64 || L == 128 || L == 256;
    return d == kTcK && l_ok && (kind == SPL_HASHER_LINEAR || h == kTcK);
}

spl_status encode_tc_launch(spl_ctx* ctx, const spl_hasher* hs, const void* x, int x_dtype,
                            uint32_t B, uint32_t m, uint32_t* codes, float* pre, cudaStream_t s) {
    if (!hs->w1_tc)
        return fail(ctx, SPL_E_DIMENSION,
                    "encode: SPL_ENCODE_TC needs d = 128 (MLP: h = 128) and L in {32, 64, 128, 256}");
    if (x_dtype != SPL_F32 && x_dtype != SPL_BF16)
        return fail(ctx, SPL_E_DIMENSION, "encode: unknown input dtype");
    if (B == 0 || m == 0) return SPL_OK;
    if (!x || !codes) return fail(ctx, SPL_E_STATE, "encode: null device pointer");
    // keys are staged with 16-byte loads (f32) / TMA (bf16), codes stored as 16-byte vectors
    if ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(codes)) % 16 != 0)
        return fail(ctx, SPL_E_DIMENSION, "encode: SPL_ENCODE_TC input and codes must be 16-byte aligned");
    TcParams prm{};
    prm.x = x;
    prm.x_bf16 = x_dtype == SPL_BF16;
    prm.H = hs->H;
    prm.m = m;
    prm.L = hs->L;
    prm.W = hs->L / 32;
    prm.linear = hs->kind == SPL_HASHER_LINEAR;
    prm.w1_tc = static_cast<const uint8_t*>(hs->w1_tc);
    prm.w2_tc = static_cast<const uint8_t*>(hs->w2_tc);
    prm.b1 = hs->b1;
    prm.codes = codes;
    prm.pre = pre;
    prm.tiles_per_problem = (m + kTcTileM - 1) / kTcTileM;
    prm.total_tiles = (uint64_t)B * hs->H * prm.tiles_per_problem;
    prm.dev_err = ctx->dev_err;
    const uint32_t N1 = prm.linear ? prm.L : kTcK;
    const size_t smem = 1024 + 3 * (size_t)tc_operand_bytes(kTcTileM) + tc_operand_bytes(N1) +
                        (prm.linear ? 0 : tc_operand_bytes(prm.L)) + kTcTileM * 8 * 4;
    const uint64_t G = std::min<uint64_t>(prm.total_tiles, (uint64_t)ctx->num_sms);
    CUtensorMap tmap;
    std::memset(&tmap, 0, sizeof(tmap));
    if (prm.x_bf16) {
        // [B*H*m rows][128] bf16, box 64 x 128 (one K block of one tile),
        // 128-byte swizzle; rows past the end are zero-filled
        static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
        if (!encode) {
            void* fn = nullptr;
            cudaDriverEntryPointQueryResult q;
            if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) !=
                    cudaSuccess ||
                q != cudaDriverEntryPointSuccess || !fn)
                return fail(ctx, SPL_E_CUDA, "encode: cuTensorMapEncodeTiled unavailable");
            encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
        }
        const cuuint64_t dims[2] = {kTcK, (cuuint64_t)B * hs->H * m};
        const cuuint64_t strides[1] = {kTcK * 2};
        const cuuint32_t box[2] = {64, kTcTileM};
        const cuuint32_t estr[2] = {1, 1};
        if (reinterpret_cast<uintptr_t>(x) % 16 != 0)
            return fail(ctx, SPL_E_DIMENSION, "encode: bf16 input must be 16-byte aligned");
        const CUresult r = encode(&tmap, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(x),
                                  dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                  CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) return fail(ctx, SPL_E_CUDA, "encode: cuTensorMapEncodeTiled failed");
    }
    // production path: MLP, bf16 keys, no pre-activation dump -> the
    // warp-specialised kernel (SPL_K2_WS=0 forces the single-team kernel)
    const char* ws_env = getenv("SPL_K2_WS");
    if (prm.x_bf16 && !prm.linear && !pre && !(ws_env && *ws_env == '0')) {
        const size_t wsmem = 1024 + (kXSlots + 1) * (size_t)tc_operand_bytes(kTcTileM) + (size_t)prm.L * 256u;
        const void* wfn = k2_ws_fn(prm.W);
        SPL_CUDA_TRY(ctx, cudaFuncSetAttribute(wfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)wsmem));
        const char* tr = getenv("SPL_K2_TRACE");
        if (tr && *tr && !stream_capturing(s)) {
            prm.trace_from = (uint32_t)atoi(tr);
            SPL_CUDA_TRY(ctx, cudaMalloc(&prm.trace, 64 * 12 * 8));
            SPL_CUDA_TRY(ctx, cudaMemsetAsync(prm.trace, 0, 64 * 12 * 8, s));
        }
        void* wargs[] = {&tmap, &prm};
        SPL_CUDA_TRY(ctx, cudaLaunchKernel(wfn, dim3((uint32_t)G), dim3(kWsThreads), wargs, wsmem, s));
        if (prm.trace) {
            // per-tile role clocks of CTA 0, relative to tile 8's GEMM1 wait (a
            // measurement aid): mma-wait-X, G1 issue, G2 wait-A1, G2 wait-D2, G2
            // issue, epi1 start, epi1 done, epi2 start
            long long h[64 * 12];
            cudaStreamSynchronize(s);
            cudaMemcpy(h, prm.trace, sizeof(h), cudaMemcpyDeviceToHost);
            cudaFree(prm.trace);
            const long long b = h[8 * 12];
            fprintf(stderr, "k2 trace (cycles, tile: x-wait g1 g2-a1wait g2-d2wait g2 e1start e1done e2start prod-wait prod-tma)\n");
            for (int i = 8; i < 24; ++i) {
                fprintf(stderr, "  %2d:", i);
                for (int k = 0; k < 10; ++k) fprintf(stderr, " %7lld", h[i * 12 + k] ? h[i * 12 + k] - b : -1);
                fprintf(stderr, "\n");
            }
            fprintf(stderr, "  period over tiles 8..56: %.0f cycles/tile\n", (double)(h[56 * 12 + 1] - h[8 * 12 + 1]) / 48);
        }
        return after_launch(ctx, "k2_encode_ws");
    }
    const void* fn = prm.x_bf16 ? k2_fn<true>(prm.W) : k2_fn<false>(prm.W);
    SPL_CUDA_TRY(ctx, cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    void* args[] = {&tmap, &prm};
    SPL_CUDA_TRY(ctx, cudaLaunchKernel(fn, dim3((uint32_t)G), dim3(kTcThreads), args, smem, s));
    return after_launch(ctx, "k2_encode_tc");
}

}  // namespace spl
