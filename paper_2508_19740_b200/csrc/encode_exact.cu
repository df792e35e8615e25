// K1 — exact-mode MLP / linear hash encoder on CUDA cores (sm_100a).
//
// Replaces mlp_forward (hashers.cpp:84-103) + sign_bits (:19-28) +
// pack_bits (bitcodes.cpp:22-41) for decode-time vectors (1 new key and 1
// query per (batch, head) per step), fused with the append into the code /
// K / V caches. Bit-exact with the reference:
//   * each output is the reference's p-ordered FMA chain
//     (matrix.hpp:92-96, contracted to vfmadd by -march=native), written as
//     __fmaf_rn so nvcc can neither reassociate nor un-fuse it;
//   * SiLU is z / (1 + expf(-z)) with every op IEEE-rounded and expf the
//     bit-exact port of glibc's (spl_expf.cuh, 0 mismatches over 2^32);
//   * packing: warp w computes columns {c*W + w : c = lane}, so word w of the
//     code is __brev(__ballot_sync(pre >= 0)) — the Appendix A.7 layout.
// The per-output chain is inherently sequential over p; parallelism is over
// (vector, output column), VT vectors per CTA share each weight load.
#include <cuda_runtime.h>
#include <stdint.h>
#include <cuda_bf16.h>

#include <string>

#include "spl_expf.cuh"
#include "spl_launch.cuh"

namespace spl {

constexpr int kEncThreads = 128;
constexpr int kVT = 8;  // vectors per CTA

struct EncParams {
    const float* w1;
    const float* b1;
    const float* w2;
    uint32_t H, d, h, L, W;
    int kind;
    uint32_t B;
    EncJob job[2];  // blockIdx.z selects the job (decode step: key append + query)
    uint32_t* dev_err;
};

__device__ __forceinline__ float silu_exact(float z) {
    const float e = spl_expf(-z);
    return __fdiv_rn(z, __fadd_rn(1.0f, e));
}

__global__ void __launch_bounds__(kEncThreads) k1_encode_exact(EncParams prm) {
    extern __shared__ float esm[];
    const EncJob& job = prm.job[blockIdx.z];
    const uint32_t head = blockIdx.y;
    const uint32_t d = prm.d, h = prm.h, L = prm.L, W = prm.W, H = prm.H;
    const uint32_t nvec = prm.B * job.m;
    const uint32_t v0 = blockIdx.x * kVT;
    if (v0 >= nvec) return;
    const uint32_t nv = min((uint32_t)kVT, nvec - v0);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    float* xs = esm;                         // [kVT][d]
    float* a1 = esm + (size_t)kVT * d;       // [kVT][h]
    __shared__ uint32_t s_bad;
    if (tid == 0) s_bad = 0;
    __syncthreads();

    // stage the inputs (zero-fill unused vector slots)
    for (uint32_t i = tid; i < kVT * d; i += kEncThreads) {
        const uint32_t v = i / d, c = i % d;
        float val = 0.0f;
        if (v < nv) {
            const uint32_t vg = v0 + v, b = vg / job.m, mi = vg % job.m;
            val = job.x[(((uint64_t)b * H + head) * job.m + mi) * d + c];
            if (!isfinite(val)) s_bad = 1;
        }
        xs[i] = val;
    }
    __syncthreads();
    if (s_bad && tid == 0) raise_dev_err(prm.dev_err, SPL_DEV_ERR_NUMERIC);

    const float* act = xs;
    uint32_t act_dim = d;
    const float* w2 = prm.w2 + (uint64_t)head * h * L;
    if (prm.kind == SPL_HASHER_MLP) {
        const float* w1 = prm.w1 + (uint64_t)head * d * h;
        const float* b1 = prm.b1 + (uint64_t)head * h;
        for (uint32_t j = tid; j < h; j += kEncThreads) {
            float acc[kVT];
#pragma unroll
            for (int v = 0; v < kVT; ++v) acc[v] = 0.0f;
#pragma unroll 4
            for (uint32_t p = 0; p < d; ++p) {
                const float w = __ldg(w1 + (uint64_t)p * h + j);
#pragma unroll
                for (int v = 0; v < kVT; ++v) acc[v] = __fmaf_rn(xs[v * d + p], w, acc[v]);
            }
            const float bj = __ldg(b1 + j);
#pragma unroll
            for (int v = 0; v < kVT; ++v) a1[v * h + j] = silu_exact(__fadd_rn(acc[v], bj));
        }
        __syncthreads();
        act = a1;
        act_dim = h;
    } else {
        w2 = prm.w1 + (uint64_t)head * d * L;  // linear: projection d x L
    }

    // layer 2 (or the linear projection) + sign + pack
    for (uint32_t w = warp; w < W; w += kEncThreads / 32) {
        const uint32_t col = lane * W + w;
        float acc[kVT];
#pragma unroll
        for (int v = 0; v < kVT; ++v) acc[v] = 0.0f;
#pragma unroll 4
        for (uint32_t p = 0; p < act_dim; ++p) {
            const float wv = __ldg(w2 + (uint64_t)p * L + col);
#pragma unroll
            for (int v = 0; v < kVT; ++v) acc[v] = __fmaf_rn(act[v * act_dim + p], wv, acc[v]);
        }
#pragma unroll
        for (int v = 0; v < kVT; ++v) {
            if ((uint32_t)v >= nv) break;
            const uint32_t vg = v0 + v, b = vg / job.m, mi = vg % job.m;
            if (job.out_mode == ENC_PRE) {
                job.pre[(((uint64_t)b * H + head) * job.m + mi) * L + col] = acc[v];
            } else {
                const uint32_t bits = __ballot_sync(0xffffffffu, acc[v] >= 0.0f);
                if (lane == 0) {
                    uint64_t row;
                    if (job.out_mode == ENC_APPEND)
                        row = ((uint64_t)b * H + head) * job.cap + (job.pos[b] - job.pos_minus_one);
                    else
                        row = ((uint64_t)b * H + head) * job.m + mi;
                    job.codes[row * W + w] = __brev(bits);
                }
            }
        }
    }

    // append: K/V rows into the caches at the same slot
    if (job.out_mode == ENC_APPEND && job.kcache) {
        for (uint32_t i = tid; i < nv * d; i += kEncThreads) {
            const uint32_t v = i / d, c = i % d;
            const uint32_t b = v0 + v;  // m == 1
            const uint64_t src = ((uint64_t)b * H + head) * d + c;
            const uint64_t dst =
                (((uint64_t)b * H + head) * job.cap + (job.pos[b] - job.pos_minus_one)) * d + c;
            const float kv = xs[v * d + c];
            const float vv = job.v_new[src];
            if (job.kv_dtype == SPL_BF16) {
                static_cast<__nv_bfloat16*>(job.kcache)[dst] = __float2bfloat16_rn(kv);
                static_cast<__nv_bfloat16*>(job.vcache)[dst] = __float2bfloat16_rn(vv);
            } else {
                static_cast<float*>(job.kcache)[dst] = kv;
                static_cast<float*>(job.vcache)[dst] = vv;
            }
        }
    }
}

spl_status encode_exact_launch(spl_ctx* ctx, const spl_hasher* hs, uint32_t B,
                               const EncJob* jobs, int njobs, cudaStream_t s) {
    EncParams prm{};
    prm.w1 = hs->w1;
    prm.b1 = hs->b1;
    prm.w2 = hs->w2;
    prm.H = hs->H;
    prm.d = hs->d;
    prm.h = hs->h;
    prm.L = hs->L;
    prm.W = hs->L / 32;
    prm.kind = hs->kind;
    prm.B = B;
    uint32_t max_m = 0;
    for (int i = 0; i < njobs; ++i) {
        prm.job[i] = jobs[i];
        max_m = jobs[i].m > max_m ? jobs[i].m : max_m;
    }
    prm.dev_err = ctx->dev_err;
    const uint32_t nvec = B * max_m;
    if (nvec == 0) return SPL_OK;
    const size_t smem = sizeof(float) * kVT * ((size_t)hs->d + (hs->kind == SPL_HASHER_MLP ? hs->h : 0));
    if (smem > 48 * 1024)
        SPL_CUDA_TRY(ctx, cudaFuncSetAttribute(k1_encode_exact,
                                               cudaFuncAttributeMaxDynamicSharedMemorySize,
                                               (int)smem));
    dim3 grid((nvec + kVT - 1) / kVT, hs->H, njobs);
    k1_encode_exact<<<grid, kEncThreads, smem, s>>>(prm);
    return after_launch(ctx, "k1_encode_exact");
}

}  // namespace spl
