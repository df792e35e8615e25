// Microbenchmark (not part of the product): what bounds the sparse-attention
// gather on this B200 — random rows of B bytes out of a large cache, L2
// flushed before every timed launch. Sweeps
//   * row size B in {256, 512, 1024} at a fixed byte total (does a wider
//     contiguous row — e.g. K and V of one token side by side — gather faster?)
//   * byte total 43 MB (config 2) and 4x that (latency vs bandwidth)
//   * access form: lane-per-row LDG.256, warp-per-row, cp.async.bulk rows
//     into a shared-memory ring (TMA 1-D), persistent grid
//   * a 67 MB contiguous stream (config-2 code scan) alone, the gather alone
//     and both at once on two streams (does the gather hide under the scan?)
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gather_sweep gather_sweep.cu
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <random>
#include <vector>

__device__ __forceinline__ void ld256(const void* p, uint32_t* w) {
    asm volatile("ld.global.nc.L1::no_allocate.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3]), "=r"(w[4]), "=r"(w[5]),
                   "=r"(w[6]), "=r"(w[7])
                 : "l"(p));
}

// lane per row, all B/32 loads of a row in flight
template <int B>
__global__ void g_lane(const uint8_t* __restrict__ base, const uint32_t* __restrict__ rows,
                       uint32_t n, uint32_t* out) {
    uint32_t acc = 0;
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const uint8_t* p = base + (uint64_t)rows[i] * B;
        uint32_t w[B / 32][8];
#pragma unroll
        for (int c = 0; c < B / 32; ++c) ld256(p + c * 32, w[c]);
#pragma unroll
        for (int c = 0; c < B / 32; ++c)
#pragma unroll
            for (int k = 0; k < 8; ++k) acc ^= w[c][k];
    }
    if (acc == 0x12345678u) out[0] = acc;
}

// warp per row: lane l reads bytes [l*B/32, (l+1)*B/32) of each of ROWS rows
template <int B, int ROWS>
__global__ void g_warp(const uint8_t* __restrict__ base, const uint32_t* __restrict__ rows,
                       uint32_t n, uint32_t* out) {
    constexpr int PL = B / 32;  // bytes per lane: 8, 16, 32
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t nw = gridDim.x * blockDim.x / 32;
    uint32_t acc = 0;
    for (uint32_t w = (blockIdx.x * blockDim.x + threadIdx.x) / 32; w * ROWS < n; w += nw) {
        const uint32_t r0 = w * ROWS;
        uint32_t v[ROWS][PL / 4];
#pragma unroll
        for (int k = 0; k < ROWS; ++k) {
            const uint32_t r = r0 + k < n ? rows[r0 + k] : rows[r0];
            const uint8_t* p = base + (uint64_t)r * B + lane * PL;
            if constexpr (PL == 8) {
                uint2 t = __ldg(reinterpret_cast<const uint2*>(p));
                v[k][0] = t.x; v[k][1] = t.y;
            } else if constexpr (PL == 16) {
                uint4 t = __ldg(reinterpret_cast<const uint4*>(p));
                v[k][0] = t.x; v[k][1] = t.y; v[k][2] = t.z; v[k][3] = t.w;
            } else {
                ld256(p, v[k]);
            }
        }
#pragma unroll
        for (int k = 0; k < ROWS; ++k)
#pragma unroll
            for (int j = 0; j < PL / 4; ++j) acc ^= v[k][j];
    }
    if (acc == 0x12345678u) out[0] = acc;
}

// cp.async.bulk: each warp's lane 0 issues DEPTH row copies into the warp's
// shared-memory stage (one mbarrier per stage), two stages per warp
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(bar)),
                 "r"(count));
}
__device__ __forceinline__ void mbar_expect(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(bar)),
                 "r"(bytes));
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
    asm volatile(
        "{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W;\n}\n" ::"r"(
            (uint32_t)__cvta_generic_to_shared(bar)),
        "r"(phase));
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            (uint32_t)__cvta_generic_to_shared(dst)),
        "l"(src), "r"(bytes), "r"((uint32_t)__cvta_generic_to_shared(bar))
        : "memory");
}

template <int B, int DEPTH>
__global__ void g_bulk(const uint8_t* __restrict__ base, const uint32_t* __restrict__ rows, uint32_t n,
                       uint32_t* out) {
    extern __shared__ __align__(128) uint8_t sm[];
    __shared__ __align__(8) uint64_t bars[8][2];
    const uint32_t warp = threadIdx.x / 32, lane = threadIdx.x & 31, nwarp = blockDim.x / 32;
    uint8_t* st = sm + (size_t)warp * 2 * DEPTH * B;
    if (lane == 0) {
        mbar_init(&bars[warp][0], 1);
        mbar_init(&bars[warp][1], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncwarp();
    const uint32_t gw = blockIdx.x * nwarp + warp, nw = gridDim.x * nwarp;
    uint32_t acc = 0;
    uint32_t ph[2] = {0, 0};
    // batch b = rows [b*DEPTH, (b+1)*DEPTH); warp takes batches gw, gw+nw, ...
    uint32_t b = gw, s = 0;
    auto issue = [&](uint32_t bb, uint32_t ss) {
        if (lane == 0 && bb * DEPTH < n) {
            const uint32_t cntr = min((uint32_t)DEPTH, n - bb * DEPTH);
            mbar_expect(&bars[warp][ss], cntr * B);
            for (uint32_t k = 0; k < cntr; ++k)
                bulk_g2s(st + (ss * DEPTH + k) * B, base + (uint64_t)rows[bb * DEPTH + k] * B, B,
                         &bars[warp][ss]);
        }
    };
    issue(b, 0);
    issue(b + nw, 1);
    while (b * DEPTH < n) {
        mbar_wait(&bars[warp][s], ph[s]);
        ph[s] ^= 1;
        const uint32_t* w = reinterpret_cast<const uint32_t*>(st + s * DEPTH * B);
        for (uint32_t k = lane; k < DEPTH * B / 4; k += 32) acc ^= w[k];
        __syncwarp();
        issue(b + 2 * nw, s);
        b += nw;
        s ^= 1;
    }
    if (acc == 0x12345678u) out[0] = acc;
}

// contiguous stream (the code scan), each CTA a chunk, 2 x 32 B per thread in flight
__global__ void __launch_bounds__(256) stream_chunk(const uint8_t* __restrict__ a, uint64_t units,
                                                    uint32_t* out) {
    const uint64_t per = (units + gridDim.x - 1) / gridDim.x;
    const uint64_t u0 = blockIdx.x * per, u1 = min(units, u0 + per);
    uint32_t acc = 0;
    for (uint64_t base = u0; base < u1; base += 4 * 256) {
        uint32_t w[4][8];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const uint64_t i = base + u * 256 + threadIdx.x;
            if (i < u1) ld256(a + i * 32, w[u]);
            else for (int k = 0; k < 8; ++k) w[u][k] = 0;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
            for (int k = 0; k < 8; ++k) acc ^= w[u][k];
    }
    if (acc == 0x12345678u) out[0] = acc;
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const uint64_t cache_bytes = 4ull << 30;
    uint8_t* buf;
    uint32_t* o;
    cudaMalloc(&buf, cache_bytes);
    cudaMalloc(&o, 4);
    cudaMemset(buf, 1, cache_bytes);
    void* flush;
    cudaMalloc(&flush, 512ull << 20);
    cudaStream_t s0, s1;
    cudaStreamCreateWithFlags(&s0, cudaStreamNonBlocking);
    cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking);
    cudaEvent_t e0, e1, e2;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventCreate(&e2);
    auto timeit = [&](const char* name, double bytes, auto launch) {
        for (int i = 0; i < 3; ++i) launch();
        cudaDeviceSynchronize();
        std::vector<float> ts;
        for (int i = 0; i < 15; ++i) {
            cudaMemsetAsync(flush, i, 512ull << 20, s0);  // evict L2, then read 256 MB so
            stream_chunk<<<sms * 3, 256, 0, s0>>>((const uint8_t*)flush, (256ull << 20) / 32, o);  // no dirty lines remain
            cudaEventRecord(e0, s0);
            launch();
            cudaEventRecord(e1, s0);
            cudaEventSynchronize(e1);
            float t;
            cudaEventElapsedTime(&t, e0, e1);
            ts.push_back(t * 1000);
        }
        // event ticks are coarse on this part (~2 us): report the mean
        float med = 0;
        for (float t : ts) med += t / ts.size();
        printf("%-44s %9.2f us  %7.1f GB/s  %s\n", name, med, bytes / (med * 1e-6) / 1e9,
               cudaGetErrorString(cudaGetLastError()));
    };
    std::mt19937 g(1);
    const double base_bytes = 2622.0 * 64 * 256;  // config 2: 32 heads x (K + V) x 2622 rows x 256 B
    for (int mult : {1, 4}) {
        for (int B : {256, 512, 1024}) {
            const uint32_t nrows = (uint32_t)(base_bytes * mult / B);
            const uint64_t cache_rows = cache_bytes / B;
            const uint32_t probs = 64;
            const uint64_t per_prob = cache_rows / probs;
            std::vector<uint32_t> rows;
            rows.reserve(nrows);
            const uint32_t take = nrows / probs;
            for (uint32_t p = 0; p < probs; ++p) {
                std::vector<uint32_t> r(take);
                for (auto& x : r) x = (uint32_t)(g() % per_prob);
                std::sort(r.begin(), r.end());
                for (auto x : r) rows.push_back((uint32_t)(p * per_prob + x));
            }
            const uint32_t n = (uint32_t)rows.size();
            uint32_t* d_rows;
            cudaMalloc(&d_rows, n * 4);
            cudaMemcpy(d_rows, rows.data(), n * 4, cudaMemcpyHostToDevice);
            const double bytes = (double)n * B;
            char nm[96];
            auto tag = [&](const char* what) {
                snprintf(nm, sizeof nm, "x%d B=%4d %s", mult, B, what);
                return nm;
            };
            timeit(tag("lane 128thr full-grid"), bytes,
                   [&] {
                       auto fl = B == 256 ? g_lane<256> : B == 512 ? g_lane<512> : g_lane<1024>;
                       fl<<<(n + 127) / 128, 128, 0, s0>>>(buf, d_rows, n, o);
                   });
            if (B == 256) {
                timeit(tag("warp rows8 full-grid"), bytes,
                       [&] { g_warp<256, 8><<<(n / 8 * 32 + 127) / 128, 128, 0, s0>>>(buf, d_rows, n, o); });
                timeit(tag("warp rows16 full-grid"), bytes,
                       [&] { g_warp<256, 16><<<(n / 16 * 32 + 127) / 128, 128, 0, s0>>>(buf, d_rows, n, o); });
                timeit(tag("warp rows16 persistent 8/SM"), bytes,
                       [&] { g_warp<256, 16><<<sms * 8, 256, 0, s0>>>(buf, d_rows, n, o); });
            } else if (B == 512) {
                timeit(tag("warp rows8 full-grid"), bytes,
                       [&] { g_warp<512, 8><<<(n / 8 * 32 + 127) / 128, 128, 0, s0>>>(buf, d_rows, n, o); });
            } else {
                timeit(tag("warp rows4 full-grid"), bytes,
                       [&] { g_warp<1024, 4><<<(n / 4 * 32 + 127) / 128, 128, 0, s0>>>(buf, d_rows, n, o); });
            }
            {
                constexpr int DEPTH = 16;
                const size_t smem = (size_t)8 * 2 * DEPTH * B;
                auto fn = B == 256 ? g_bulk<256, DEPTH> : B == 512 ? g_bulk<512, DEPTH> : g_bulk<1024, DEPTH>;
                if (smem <= 200 * 1024) {
                    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
                    timeit(tag("bulk 8 warps x2x16 rows, 1 CTA/SM"), bytes,
                           [&] { fn<<<sms, 256, smem, s0>>>(buf, d_rows, n, o); });
                }
                const size_t smem4 = (size_t)4 * 2 * DEPTH * B;
                if (smem4 <= 100 * 1024) {
                    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem4);
                    timeit(tag("bulk 4 warps x2x16 rows, 2 CTA/SM"), bytes,
                           [&] { fn<<<sms * 2, 128, smem4, s0>>>(buf, d_rows, n, o); });
                }
            }
            if (mult == 1 && B == 256) {
                // scan + gather concurrency
                const uint64_t units = (67108864ull) / 32;  // 67 MB of codes
                uint8_t* scan = buf + (3ull << 30);
                timeit("stream 67MB alone (444 CTAs)", 67108864.0,
                       [&] { stream_chunk<<<444, 256, 0, s0>>>(scan, units, o); });
                timeit("stream 67MB + gather 43MB, two streams", 67108864.0 + bytes, [&] {
                    cudaEventRecord(e2, s0);
                    cudaStreamWaitEvent(s1, e2, 0);
                    g_warp<256, 16><<<sms * 4, 256, 0, s1>>>(buf, d_rows, n, o);
                    stream_chunk<<<444, 256, 0, s0>>>(scan, units, o);
                    cudaEventRecord(e2, s1);
                    cudaStreamWaitEvent(s0, e2, 0);
                });
                timeit("stream then gather, one stream", 67108864.0 + bytes, [&] {
                    stream_chunk<<<444, 256, 0, s0>>>(scan, units, o);
                    g_warp<256, 16><<<(n / 16 * 32 + 127) / 128, 128, 0, s0>>>(buf, d_rows, n, o);
                });
            }
            cudaFree(d_rows);
        }
    }
    return 0;
}
