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
#include <cuda_bf16.h>

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
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[16]) {
    uint32_t r[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
          "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
          "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
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

__global__ void __launch_bounds__(kTcThreads, 1) k2_encode_tc(TcParams prm) {
    extern __shared__ uint8_t smem_raw[];
    __shared__ __align__(8) uint64_t s_bar[2];
    __shared__ uint32_t s_tmem;
    __shared__ float s_b1[kTcK];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t L = prm.L, W = prm.W;
    const uint32_t N1 = prm.linear ? L : kTcK;
    // 1024-aligned operand regions: sX, sA1 (128 rows), sW1 (N1 rows), sW2 (L rows), s_code
    const uint32_t base_s = (smem_u32(smem_raw) + 1023u) & ~1023u;
    uint8_t* base = smem_raw + (base_s - smem_u32(smem_raw));
    uint8_t* sX = base;
    uint8_t* sA1 = sX + tc_operand_bytes(kTcTileM);
    uint8_t* sW1 = sA1 + tc_operand_bytes(kTcTileM);
    uint8_t* sW2 = sW1 + tc_operand_bytes(N1);
    uint32_t* s_code = reinterpret_cast<uint32_t*>(sW2 + (prm.linear ? 0u : tc_operand_bytes(L)));

    const uint64_t T = prm.total_tiles;
    const uint64_t t0 = T * blockIdx.x / gridDim.x, t1 = T * (blockIdx.x + 1) / gridDim.x;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                         smem_u32(&s_tmem))
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&s_bar[0])));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&s_bar[1])));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    fence_before();
    __syncthreads();
    fence_after();
    const uint32_t tmem = s_tmem;
    const uint32_t tD1 = tmem, tD2 = tmem + kTcK;
    const uint32_t quarter = (uint32_t)(warp & 3), half = (uint32_t)(warp >> 2);
    const uint32_t row = quarter * 32 + lane;  // this thread's TMEM lane = tile row
    const uint32_t lane_addr = (quarter * 32) << 16;

    uint32_t phase = 0;
    uint64_t cur_head = ~0ull;
    if (t0 < t1) {
        const uint64_t bh0 = t0 / prm.tiles_per_problem;
        stage_x(prm, bh0, (uint32_t)(t0 % prm.tiles_per_problem) * kTcTileM, sX);
    }
    for (uint64_t t = t0; t < t1; ++t) {
        const uint64_t bh = t / prm.tiles_per_problem;
        const uint32_t row0 = (uint32_t)(t % prm.tiles_per_problem) * kTcTileM;
        const uint64_t head = bh % prm.H;
        if (head != cur_head) {  // previous MMAs are complete (waited below)
            const uint4* g1 = reinterpret_cast<const uint4*>(prm.w1_tc + head * tc_operand_bytes(N1));
            for (uint32_t i = tid; i < tc_operand_bytes(N1) / 16; i += kTcThreads)
                reinterpret_cast<uint4*>(sW1)[i] = __ldg(g1 + i);
            if (!prm.linear) {
                const uint4* g2 = reinterpret_cast<const uint4*>(prm.w2_tc + head * tc_operand_bytes(L));
                for (uint32_t i = tid; i < tc_operand_bytes(L) / 16; i += kTcThreads)
                    reinterpret_cast<uint4*>(sW2)[i] = __ldg(g2 + i);
                for (uint32_t i = tid; i < kTcK; i += kTcThreads) s_b1[i] = prm.b1[head * kTcK + i];
            }
            cur_head = head;
        }
        fence_async_smem();
        fence_before();
        __syncthreads();
        // ---- GEMM1
        if (tid == 0) {
            fence_after();
            gemm_k128(tD1, smem_u32(sX), smem_u32(sW1), N1);
            umma_commit(&s_bar[0]);
        }
        mbar_wait(&s_bar[0], phase);
        fence_after();
        uint32_t tZ = tD1;
        if (!prm.linear) {
            // ---- epilogue 1: +b1, SiLU -> bf16 A1 (columns [64 half, +64))
#pragma unroll 1
            for (uint32_t c0 = half * 64; c0 < half * 64 + 64; c0 += 16) {
                float v[16];
                tmem_ld16(tD1 + lane_addr + c0, v);
                uint32_t p[8];
#pragma unroll
                for (int i = 0; i < 16; i += 2) {
                    const float z0 = v[i] + s_b1[c0 + i], z1 = v[i + 1] + s_b1[c0 + i + 1];
                    p[i / 2] = pack_bf16(__fdividef(z0, 1.0f + __expf(-z0)),
                                         __fdividef(z1, 1.0f + __expf(-z1)));
                }
                *reinterpret_cast<uint4*>(sA1 + tc_sw_off(row, c0, kTcTileM)) =
                    make_uint4(p[0], p[1], p[2], p[3]);
                *reinterpret_cast<uint4*>(sA1 + tc_sw_off(row, c0 + 8, kTcTileM)) =
                    make_uint4(p[4], p[5], p[6], p[7]);
            }
            fence_async_smem();
            fence_before();
            __syncthreads();
            // ---- GEMM2
            if (tid == 0) {
                fence_after();
                gemm_k128(tD2, smem_u32(sA1), smem_u32(sW2), L);
                umma_commit(&s_bar[1]);
            }
            tZ = tD2;
        }
        // sX is free (GEMM1 has completed): stage the next tile's keys while
        // GEMM2 runs
        if (t + 1 < t1) {
            const uint64_t nbh = (t + 1) / prm.tiles_per_problem;
            stage_x(prm, nbh, (uint32_t)((t + 1) % prm.tiles_per_problem) * kTcTileM, sX);
        }
        if (!prm.linear) {
            mbar_wait(&s_bar[1], phase);
            fence_after();
        }
        // ---- epilogue 2: sign bits of columns [half L/2, +L/2) -> partial words
        uint32_t wd[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        const uint32_t grow = row0 + row;
#pragma unroll 1
        for (uint32_t c0 = half * (L / 2); c0 < (half + 1) * (L / 2); c0 += 16) {
            float v[16];
            tmem_ld16(tZ + lane_addr + c0, v);
#pragma unroll
            for (int i = 0; i < 16; ++i) {
                const uint32_t j = c0 + i;  // W divides 16: word j % W = i % W
                const uint32_t bit = v[i] >= 0.0f ? 1u : 0u;
                if (W == 1) wd[0] |= bit << (31 - j);
                else if (W == 2) wd[i & 1] |= bit << (31 - (j >> 1));
                else if (W == 4) wd[i & 3] |= bit << (31 - (j >> 2));
                else wd[i & 7] |= bit << (31 - (j >> 3));
            }
            if (prm.pre && grow < prm.m)
                for (int i = 0; i < 16; ++i) prm.pre[((bh * prm.m) + grow) * L + c0 + i] = v[i];
        }
        if (half == 1)
            for (uint32_t w = 0; w < W; ++w) s_code[row * 8 + w] = wd[w];
        fence_before();
        __syncthreads();
        if (half == 0 && grow < prm.m) {
            uint32_t* dst = prm.codes + ((bh * prm.m) + grow) * W;
            if (W == 4) {
                *reinterpret_cast<uint4*>(dst) =
                    make_uint4(wd[0] | s_code[row * 8 + 0], wd[1] | s_code[row * 8 + 1],
                               wd[2] | s_code[row * 8 + 2], wd[3] | s_code[row * 8 + 3]);
            } else {
                for (uint32_t w = 0; w < W; ++w) dst[w] = wd[w] | s_code[row * 8 + w];
            }
        }
        phase ^= 1u;
    }
    fence_before();
    __syncthreads();
    fence_after();
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
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
    const size_t smem = 1024 + 2 * (size_t)tc_operand_bytes(kTcTileM) + tc_operand_bytes(N1) +
                        (prm.linear ? 0 : tc_operand_bytes(prm.L)) + kTcTileM * 8 * 4;
    SPL_CUDA_TRY(ctx, cudaFuncSetAttribute(k2_encode_tc, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)smem));
    const uint64_t G = std::min<uint64_t>(prm.total_tiles, (uint64_t)ctx->num_sms);
    k2_encode_tc<<<(uint32_t)G, kTcThreads, smem, s>>>(prm);
    return after_launch(ctx, "k2_encode_tc");
}

}  // namespace spl
