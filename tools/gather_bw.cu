// Microbenchmark (not part of the product): HBM bandwidth of the sparse-
// attention access pattern — gather R random rows of B bytes out of a large
// K (or V) cache, ascending row ids per problem like a top-k list.
//   lane : lane-per-row, each lane streams its row with 16-byte loads
//   warp : warp-per-row, each lane one 8-byte slice (B = 256)
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gather_bw gather_bw.cu
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <random>
#include <cuda_runtime.h>

template <int B, int INFL>
__global__ void g_lane(const uint4* __restrict__ base, const uint32_t* __restrict__ rows, uint32_t n, uint32_t* out) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    uint32_t acc = 0;
    if (i < n) {
        const uint4* p = base + (uint64_t)rows[i] * (B / 16);
#pragma unroll
        for (int c = 0; c < B / 16; c += INFL) {
            uint4 v[INFL];
#pragma unroll
            for (int k = 0; k < INFL; ++k) v[k] = __ldg(p + c + k);
#pragma unroll
            for (int k = 0; k < INFL; ++k) acc ^= v[k].x ^ v[k].y ^ v[k].z ^ v[k].w;
        }
    }
    if (acc == 0x12345678u) out[0] = acc;
}

__device__ __forceinline__ void ld256nc(const void* p, uint32_t* w) {
    asm volatile("ld.global.nc.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3]), "=r"(w[4]), "=r"(w[5]), "=r"(w[6]), "=r"(w[7])
                 : "l"(p));
}
template <int B>
__global__ void g_lane32(const uint8_t* __restrict__ base, const uint32_t* __restrict__ rows, uint32_t n, uint32_t* out) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    uint32_t acc = 0;
    if (i < n) {
        const uint8_t* p = base + (uint64_t)rows[i] * B;
        uint32_t w[B / 32][8];
#pragma unroll
        for (int c = 0; c < B / 32; ++c) ld256nc(p + c * 32, w[c]);
#pragma unroll
        for (int c = 0; c < B / 32; ++c)
#pragma unroll
            for (int k = 0; k < 8; ++k) acc ^= w[c][k];
    }
    if (acc == 0x12345678u) out[0] = acc;
}

template <int ROWS>
__global__ void g_warp(const uint2* __restrict__ base, const uint32_t* __restrict__ rows, uint32_t n, uint32_t* out) {
    const uint32_t w = (blockIdx.x * blockDim.x + threadIdx.x) / 32, lane = threadIdx.x & 31;
    uint32_t acc = 0;
    const uint32_t r0 = w * ROWS;
    uint2 v[ROWS];
#pragma unroll
    for (int k = 0; k < ROWS; ++k)
        if (r0 + k < n) v[k] = __ldg(base + (uint64_t)rows[r0 + k] * 32 + lane); else v[k] = make_uint2(0, 0);
#pragma unroll
    for (int k = 0; k < ROWS; ++k) acc ^= v[k].x ^ v[k].y;
    if (acc == 0x12345678u) out[0] = acc;
}

int main() {
    const uint64_t cache_rows = 32ull * 131072;  // 32 heads x 128K rows
    const uint32_t k = 2622 * 32 * 2;              // config 2: K and V rows of 32 heads
    for (int B : {256, 512}) {
        uint8_t* buf; uint32_t* d_rows; uint32_t* o;
        cudaMalloc(&buf, cache_rows * B); cudaMalloc(&o, 4);
        cudaMemset(buf, 1, cache_rows * B);
        std::vector<uint32_t> rows(k);
        std::mt19937 g(1);
        for (uint32_t h = 0; h < 64; ++h) {  // 64 problems (32 K + 32 V), 2% of 128K each, ascending
            std::vector<uint32_t> r(131072);
            for (uint32_t i = 0; i < 131072; ++i) r[i] = i;
            std::shuffle(r.begin(), r.end(), g);
            std::sort(r.begin(), r.begin() + 2622);
            for (uint32_t i = 0; i < 2622; ++i) rows[h * 2622 + i] = (h % 32) * 131072 + r[i];
        }
        cudaMalloc(&d_rows, k * 4);
        cudaMemcpy(d_rows, rows.data(), k * 4, cudaMemcpyHostToDevice);
        cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
        void* flush; cudaMalloc(&flush, 512ull << 20);
        auto timeit = [&](const char* name, auto launch) {
            for (int i = 0; i < 3; ++i) launch();
            float ms = 0;
            for (int i = 0; i < 10; ++i) {
                cudaMemset(flush, i, 512ull << 20);  // evict L2
                cudaEventRecord(e0);
                launch();
                cudaEventRecord(e1); cudaEventSynchronize(e1);
                float t; cudaEventElapsedTime(&t, e0, e1); ms += t;
            }
            ms /= 10;
            printf("B=%d %-22s %8.2f us  %7.1f GB/s  %s\n", B, name, ms * 1000, (double)k * B / (ms * 1e-3) / 1e9,
                   cudaGetErrorString(cudaGetLastError()));
        };
        if (B == 256) {
            timeit("lane infl4 tpb128", [&] { g_lane<256, 4><<<(k + 127) / 128, 128>>>((const uint4*)buf, d_rows, k, o); });
            timeit("lane infl8 tpb128", [&] { g_lane<256, 8><<<(k + 127) / 128, 128>>>((const uint4*)buf, d_rows, k, o); });
            timeit("lane infl16 tpb128", [&] { g_lane<256, 16><<<(k + 127) / 128, 128>>>((const uint4*)buf, d_rows, k, o); });
            timeit("lane infl16 tpb64", [&] { g_lane<256, 16><<<(k + 63) / 64, 64>>>((const uint4*)buf, d_rows, k, o); });
            timeit("lane32B tpb128", [&] { g_lane32<256><<<(k + 127) / 128, 128>>>(buf, d_rows, k, o); });
            timeit("lane32B tpb64", [&] { g_lane32<256><<<(k + 63) / 64, 64>>>(buf, d_rows, k, o); });
            timeit("warp rows8", [&] { g_warp<8><<<(k / 8 * 32 + 127) / 128, 128>>>((const uint2*)buf, d_rows, k, o); });
            timeit("warp rows16", [&] { g_warp<16><<<(k / 16 * 32 + 127) / 128, 128>>>((const uint2*)buf, d_rows, k, o); });
            timeit("warp rows32", [&] { g_warp<32><<<(k / 32 * 32 + 127) / 128, 128>>>((const uint2*)buf, d_rows, k, o); });
        } else {
            timeit("lane infl8 tpb128", [&] { g_lane<512, 8><<<(k + 127) / 128, 128>>>((const uint4*)buf, d_rows, k, o); });
            timeit("lane infl16 tpb128", [&] { g_lane<512, 16><<<(k + 127) / 128, 128>>>((const uint4*)buf, d_rows, k, o); });
            timeit("lane32B tpb128", [&] { g_lane32<512><<<(k + 127) / 128, 128>>>(buf, d_rows, k, o); });
        }
        cudaFree(flush);
        cudaFree(buf); cudaFree(d_rows); cudaFree(o);
    }
    return 0;
}
