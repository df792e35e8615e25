// Probe (not part of the product): how does tcgen05.mma kind::f16 with an
// F16 accumulator lay D out in TMEM, and does reading it cost fewer TMEM
// bytes than an F32 accumulator? One CTA, M = 128, N = 256, K = 128 (8 MMAs),
// A = B-independent patterns so every D element is distinct; the raw 32-bit
// TMEM words of columns 0..255 are dumped for rows 0..127 and decoded on the
// host. Also times a 32x32b.x16 read sweep of 256 columns for both formats.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tmem_f16_probe tmem_f16_probe.cu
#include <cuda_fp16.h>
#include <cstdio>
#include <cstdint>
#include <cstring>
#include <vector>
#include <cmath>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
// K-major, SWIZZLE_128B operand: element (r, k) of a rows x 128 operand
__host__ __device__ inline uint32_t sw_off(uint32_t r, uint32_t k, uint32_t rows) {
    const uint32_t kb = k >> 6, kk = k & 63u;
    return kb * rows * 128u + r * 128u + ((((kk >> 3) ^ (r & 7u)) & 7u) << 4) + ((kk & 7u) << 1);
}
__device__ inline uint64_t desc(uint32_t saddr) {
    return (uint64_t)((saddr >> 4) & 0x3FFFu) | (1ull << 16) | ((uint64_t)(1024u >> 4) << 32) | (1ull << 46) | (2ull << 61);
}
// kind::f16 idesc: D fmt bits [4,6): 0 = f16, 1 = f32; A fmt [7,10): 0 = f16, 1 = bf16; B fmt [10,13)
__device__ inline uint32_t idesc(uint32_t N, bool d_f32) {
    return ((d_f32 ? 1u : 0u) << 4) | (0u << 7) | (0u << 10) | ((N >> 3) << 17) | ((128u >> 4) << 24);
}

template <bool DF32>
__global__ void probe(const __half* A, const __half* B, uint32_t* dump, long long* cycles) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint32_t s_tmem;
    __shared__ __align__(8) uint64_t bar;
    uint8_t* sA = sm;             // 128 x 128 f16 = 32 KB
    uint8_t* sB = sm + 32768;     // 256 x 128 f16 = 64 KB
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    for (int i = tid; i < 128 * 128; i += blockDim.x) {
        const int r = i / 128, k = i % 128;
        *reinterpret_cast<__half*>(sA + sw_off(r, k, 128)) = A[i];
    }
    for (int i = tid; i < 256 * 128; i += blockDim.x) {
        const int r = i / 128, k = i % 128;
        *reinterpret_cast<__half*>(sB + sw_off(r, k, 256)) = B[i];
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&s_tmem)) : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = s_tmem;
    if (tid == 0) {
        const uint32_t id = idesc(256, DF32);
        for (uint32_t s = 0; s < 8; ++s) {
            const uint64_t da = desc(smem_u32(sA) + (s >> 2) * 128u * 128u + (s & 3u) * 32u);
            const uint64_t db = desc(smem_u32(sB) + (s >> 2) * 256u * 128u + (s & 3u) * 32u);
            asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                         "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem),
                         "l"(da), "l"(db), "r"(id), "r"(s > 0 ? 1u : 0u));
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)) : "memory");
    }
    uint32_t done = 0;
    while (!done)
        asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0, 1, 0, p; }"
                     : "=r"(done) : "r"(smem_u32(&bar)) : "memory");
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t row = (warp & 3) * 32 + lane;
    const uint32_t taddr = tmem + (((warp & 3) * 32) << 16);
    if (warp < 4) {
        for (uint32_t c0 = 0; c0 < 256; c0 += 16) {
            uint32_t r[16];
            asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                         : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                           "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
                         : "r"(taddr + c0));
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            for (int i = 0; i < 16; ++i) dump[row * 256 + c0 + i] = r[i];
        }
        // read-throughput sweep: 64 passes over 128 (f16) or 256 (f32) columns
        const uint32_t ncol = DF32 ? 256 : 128;
        __syncwarp();
        const long long t0 = clock64();
        uint32_t acc = 0;
        for (int pass = 0; pass < 64; ++pass)
            for (uint32_t c0 = 0; c0 < ncol; c0 += 32) {
                uint32_t r[32];
                asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                             : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                               "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
                               "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
                               "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
                             : "r"(taddr + c0));
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                for (int i = 0; i < 32; ++i) acc ^= r[i];
            }
        const long long t1 = clock64();
        if (lane == 0) cycles[warp] = t1 - t0;
        if (acc == 0x12345678u) dump[0] = acc;
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
}

int main() {
    // A[m][k] = (m == k) ? 1 : 0 (128 x 128), B[n][k] = small distinct values
    // -> D[m][n] = B[n][m] for m < 128
    std::vector<__half> A(128 * 128), B(256 * 128);
    for (int m = 0; m < 128; ++m)
        for (int k = 0; k < 128; ++k) A[m * 128 + k] = __float2half(m == k ? 1.0f : 0.0f);
    for (int n = 0; n < 256; ++n)
        for (int k = 0; k < 128; ++k) B[n * 128 + k] = __float2half((float)((n * 7 + k * 3) % 97) / 8.0f - 5.0f);
    __half *dA, *dB;
    uint32_t* dd;
    long long* dc;
    cudaMalloc(&dA, A.size() * 2);
    cudaMalloc(&dB, B.size() * 2);
    cudaMalloc(&dd, 128 * 256 * 4);
    cudaMalloc(&dc, 8 * 8);
    cudaMemcpy(dA, A.data(), A.size() * 2, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, B.data(), B.size() * 2, cudaMemcpyHostToDevice);
    for (int f32 = 0; f32 < 2; ++f32) {
        auto fn = f32 ? probe<true> : probe<false>;
        cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, 98304 + 1024);
        cudaMemset(dd, 0, 128 * 256 * 4);
        fn<<<1, 128, 98304 + 1024>>>(dA, dB, dd, dc);
        cudaError_t e = cudaDeviceSynchronize();
        std::vector<uint32_t> h(128 * 256);
        long long cyc[4];
        cudaMemcpy(h.data(), dd, h.size() * 4, cudaMemcpyDeviceToHost);
        cudaMemcpy(cyc, dc, sizeof(cyc), cudaMemcpyDeviceToHost);
        printf("== D %s  (%s)\n", f32 ? "f32" : "f16", cudaGetErrorString(e));
        // expected D[m][n] = B[n][m]
        auto expect = [&](int m, int n) { return __half2float(B[n * 128 + m]); };
        for (int m : {0, 1, 5}) {
            printf("row %d:", m);
            for (int c = 0; c < 6; ++c) {
                const uint32_t w = h[m * 256 + c];
                if (f32) {
                    float f; memcpy(&f, &w, 4);
                    printf(" c%d=%.3f(exp n%d=%.3f)", c, f, c, expect(m, c));
                } else {
                    __half lo, hi; uint16_t l = w & 0xffff, u = w >> 16;
                    memcpy(&lo, &l, 2); memcpy(&hi, &u, 2);
                    printf(" c%d=[%.3f|%.3f]", c, __half2float(lo), __half2float(hi));
                }
            }
            printf("\n");
            if (!f32) {
                printf("   expected n0..5:");
                for (int n = 0; n < 6; ++n) printf(" %.3f", expect(m, n));
                printf("  n128..130: %.3f %.3f %.3f\n", expect(m, 128), expect(m, 129), expect(m, 130));
            }
        }
        printf("read sweep: %lld cycles/warp for 64 x %d cols x 32 lanes x 4 B -> %.1f B/clk/warp\n", cyc[0],
               f32 ? 256 : 128, 64.0 * (f32 ? 256 : 128) * 32 * 4 / (double)cyc[0]);
    }
    return 0;
}
