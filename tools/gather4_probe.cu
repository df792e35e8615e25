// Probe (not part of the product): random-row gathers of a bf16 K cache
// ([rows][128] bf16 = 256-byte rows) by TMA tile::gather4 (4 rows per
// instruction into shared memory, mbarrier completion) vs warp-per-row
// register loads, as device time per call after an L2 flush (graph of N x
// (flush, kernel) minus N x flush). 2622 x 64 rows = 43 MB, as the config-2
// decode step's K and V gathers.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gather4_probe gather4_probe.cu -lcuda
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <functional>
#include <random>
#include <vector>

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// each CTA gathers `per` rows (multiple of 4) in rounds of `ring` rows
template <int RING>
__global__ void __launch_bounds__(128) g4(const __grid_constant__ CUtensorMap tm, const int* rows, uint32_t n,
                                          uint32_t per, uint32_t* out) {
    extern __shared__ __align__(1024) uint8_t buf[];
    __shared__ __align__(8) uint64_t bar;
    const uint32_t r0 = blockIdx.x * per, r1 = min(n, r0 + per);
    if (r0 >= r1) return;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    uint32_t phase = 0, acc = 0;
    for (uint32_t b = r0; b < r1; b += RING) {
        const uint32_t cnt = min((uint32_t)RING, r1 - b);  // multiple of 4
        if (threadIdx.x == 0) {
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&bar)), "r"(cnt * 256)
                         : "memory");
            for (uint32_t i = 0; i < cnt; i += 4) {
                asm volatile(
                    "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
                    " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(sa(buf + i * 256)),
                    "l"(reinterpret_cast<uint64_t>(&tm)), "r"(0), "r"(rows[b + i]), "r"(rows[b + i + 1]),
                    "r"(rows[b + i + 2]), "r"(rows[b + i + 3]), "r"(sa(&bar))
                    : "memory");
            }
        }
        uint32_t done = 0;
        while (!done)
            asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                         : "=r"(done) : "r"(sa(&bar)), "r"(phase) : "memory");
        phase ^= 1;
        acc ^= reinterpret_cast<const uint32_t*>(buf)[threadIdx.x];
        __syncthreads();
    }
    if (acc == 0x12345678u) out[0] = acc;
}

template <int R>
__global__ void g_warp(const uint8_t* __restrict__ base, const int* __restrict__ rows, uint32_t n, uint32_t* out) {
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t w = (blockIdx.x * blockDim.x + threadIdx.x) / 32;
    uint32_t acc = 0;
    if (w * R < n) {
        uint2 v[R];
#pragma unroll
        for (int k = 0; k < R; ++k) {
            const uint32_t r = w * R + k < n ? rows[w * R + k] : rows[w * R];
            v[k] = __ldg(reinterpret_cast<const uint2*>(base + (uint64_t)r * 256) + lane);
        }
#pragma unroll
        for (int k = 0; k < R; ++k) acc ^= v[k].x ^ v[k].y;
    }
    if (acc == 0x12345678u) out[0] = acc;
}
__global__ void stream_rd(const uint4* a, uint64_t n, uint32_t* out) {
    uint32_t acc = 0;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        acc ^= __ldcg(a + i).x;
    if (acc == 0x12345678u) out[0] = acc;
}

int main() {
    const uint64_t ROWS = 64ull * 131072;  // 64 caches of 131072 rows (K and V of 32 heads)
    uint8_t *kv, *flush;
    uint32_t* o;
    int* d_rows;
    cudaMalloc(&kv, ROWS * 256);
    cudaMalloc(&flush, 512ull << 20);
    cudaMalloc(&o, 4);
    cudaMemset(kv, 1, ROWS * 256);
    const uint32_t kk = 2624, P = 64;  // multiple of 4 per problem
    std::vector<int> rows(kk * P);
    std::mt19937 g(3);
    for (uint32_t p = 0; p < P; ++p) {
        std::vector<int> r(kk);
        for (auto& x : r) x = (int)(p * 131072u + g() % 131072u);
        std::sort(r.begin(), r.end());
        std::copy(r.begin(), r.end(), rows.begin() + p * kk);
    }
    const uint32_t n = kk * P;
    cudaMalloc(&d_rows, n * 4);
    cudaMemcpy(d_rows, rows.data(), n * 4, cudaMemcpyHostToDevice);
    // tensor map: [ROWS][128] bf16, box {128, 1} (gather4 takes 4 row coordinates)
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    auto encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    CUtensorMap tm;
    const cuuint64_t dims[2] = {128, ROWS};
    const cuuint64_t strides[1] = {256};
    const cuuint32_t box[2] = {128, 1};
    const cuuint32_t estr[2] = {1, 1};
    CUresult r = encode(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, kv, dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("tensor map: %d\n", (int)r);
    cudaStream_t s;
    cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    auto flush_l2 = [&]() {
        cudaMemsetAsync(flush, 7, 512ull << 20, s);
        stream_rd<<<592, 256, 0, s>>>((const uint4*)flush, (256ull << 20) / 16, o);
    };
    const int N = 20;
    auto graph_us = [&](std::function<void()> body) {
        cudaGraph_t gr;
        cudaGraphExec_t ge;
        cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
        for (int i = 0; i < N; ++i) body();
        cudaStreamEndCapture(s, &gr);
        cudaGraphInstantiate(&ge, gr, 0);
        float best = 1e30f;
        for (int t = 0; t < 4; ++t) {
            cudaGraphLaunch(ge, s);
            cudaStreamSynchronize(s);
            cudaEventRecord(e0, s);
            cudaGraphLaunch(ge, s);
            cudaEventRecord(e1, s);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            best = std::min(best, ms);
        }
        cudaGraphExecDestroy(ge);
        cudaGraphDestroy(gr);
        return best * 1000.0 / N;
    };
    const double base = graph_us([&] { flush_l2(); });
    const double bytes = (double)n * 256;
    auto run = [&](const char* name, std::function<void()> fn2) {
        const double t = graph_us([&] { flush_l2(); fn2(); }) - base;
        printf("%-52s %8.2f us  %7.1f GB/s  %s\n", name, t, bytes / t / 1e3, cudaGetErrorString(cudaGetLastError()));
    };
    run("warp x 8 rows (registers)", [&] { g_warp<8><<<(n / 8 * 32 + 127) / 128, 128, 0, s>>>(kv, d_rows, n, o); });
    for (uint32_t per : {64u, 128u, 256u}) {
        char nm[96];
        snprintf(nm, sizeof nm, "gather4, %u rows per CTA, ring 64 rows", per);
        cudaFuncSetAttribute(g4<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 256);
        run(nm, [&] { g4<64><<<(n + per - 1) / per, 128, 64 * 256, s>>>(tm, d_rows, n, per, o); });
        snprintf(nm, sizeof nm, "gather4, %u rows per CTA, ring 128 rows", per);
        cudaFuncSetAttribute(g4<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, 128 * 256);
        run(nm, [&] { g4<128><<<(n + per - 1) / per, 128, 128 * 256, s>>>(tm, d_rows, n, per, o); });
    }
    return 0;
}
