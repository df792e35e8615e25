// Microbenchmark (not part of the product): the config-2 decode step's memory
// phases timed as device time per call with L2 flushed before each call —
// a CUDA graph of N x (flush, kernel) minus a graph of N x flush, so launch
// overhead is excluded (single-launch CUDA-event timing on this box carries
// ~6 us of launch latency, tools/cold_probe.cu "empty kernel").
//   stream   : 67 MB contiguous code stream (444 CTAs x 256 threads, LDG.256)
//   gather   : 2622 random rows x 64 (K and V of 32 heads), 256-byte rows
//   gather512: 2622 random rows x 32, 512-byte rows (K|V interleaved per token)
//   spin+pf  : a 7 us "encoder" kernel that first issues cp.async.bulk.prefetch.L2
//              of the whole code cache, then the stream
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o step_probe step_probe.cu
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <functional>
#include <random>
#include <vector>

__device__ __forceinline__ void ld256(const void* p, uint32_t* w) {
    asm volatile("ld.global.nc.L1::no_allocate.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3]), "=r"(w[4]), "=r"(w[5]),
                   "=r"(w[6]), "=r"(w[7])
                 : "l"(p));
}
__global__ void __launch_bounds__(256) stream_chunk(const uint8_t* __restrict__ a, uint64_t units,
                                                    uint32_t* out, int selfpf = 0) {
    const uint64_t per = (units + gridDim.x - 1) / gridDim.x;
    const uint64_t u0 = blockIdx.x * per, u1 = min(units, u0 + per);
    if (selfpf && threadIdx.x == 0)
        for (uint64_t b = u0 * 32; b < u1 * 32; b += 32768) {
            const uint32_t n = (uint32_t)min((uint64_t)32768, u1 * 32 - b) & ~15u;
            if (n) asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a + b), "r"(n) : "memory");
        }
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
// warp per row, R rows in flight per warp, row = 32 lanes x (B/32) bytes
template <int B, int R>
__global__ void g_warp(const uint8_t* __restrict__ base, const uint32_t* __restrict__ rows, uint32_t n,
                       uint32_t* out) {
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t w = (blockIdx.x * blockDim.x + threadIdx.x) / 32;
    uint32_t acc = 0;
    if (w * R < n) {
        if constexpr (B == 256) {
            uint2 v[R];
#pragma unroll
            for (int k = 0; k < R; ++k) {
                const uint32_t r = w * R + k < n ? rows[w * R + k] : rows[w * R];
                v[k] = __ldg(reinterpret_cast<const uint2*>(base + (uint64_t)r * B) + lane);
            }
#pragma unroll
            for (int k = 0; k < R; ++k) acc ^= v[k].x ^ v[k].y;
        } else {
            uint4 v[R];
#pragma unroll
            for (int k = 0; k < R; ++k) {
                const uint32_t r = w * R + k < n ? rows[w * R + k] : rows[w * R];
                v[k] = __ldg(reinterpret_cast<const uint4*>(base + (uint64_t)r * B) + lane);
            }
#pragma unroll
            for (int k = 0; k < R; ++k) acc ^= v[k].x ^ v[k].y ^ v[k].z ^ v[k].w;
        }
    }
    if (acc == 0x12345678u) out[0] = acc;
}
__global__ void spin_pf(const uint8_t* a, uint64_t bytes, uint32_t ns, int pf) {
    if (pf == 2) {  // every thread prefetches 128-byte lines of the CTA's share
        const uint64_t per = ((bytes + gridDim.x - 1) / gridDim.x + 127) & ~127ull;
        const uint64_t b0 = blockIdx.x * per, b1 = min(bytes, b0 + per);
        for (uint64_t b = b0 + threadIdx.x * 128ull; b < b1; b += blockDim.x * 128ull)
            asm volatile("prefetch.global.L2 [%0];" ::"l"(a + b));
    }
    if (pf == 3) {  // every thread loads 16 B per 128-byte line (data lands in L2), discarded
        const uint64_t per = ((bytes + gridDim.x - 1) / gridDim.x + 127) & ~127ull;
        const uint64_t b0 = blockIdx.x * per, b1 = min(bytes, b0 + per);
        uint32_t acc = 0;
        for (uint64_t b = b0 + threadIdx.x * 128ull; b < b1; b += blockDim.x * 128ull * 4) {
            uint32_t v[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const uint64_t bb = b + u * blockDim.x * 128ull;
                v[u] = bb < b1 ? __ldcg(reinterpret_cast<const uint32_t*>(a + bb)) : 0u;
            }
            acc ^= v[0] ^ v[1] ^ v[2] ^ v[3];
        }
        if (acc == 0x12345678u) *(volatile uint32_t*)nullptr = acc;
    }
    if (pf == 1 && threadIdx.x == 0) {
        const uint64_t per = ((bytes + gridDim.x - 1) / gridDim.x + 15) & ~15ull;
        const uint64_t b0 = blockIdx.x * per, b1 = min(bytes, b0 + per);
        for (uint64_t b = b0; b < b1; b += 32768) {
            const uint32_t n = (uint32_t)min((uint64_t)32768, b1 - b) & ~15u;
            if (n) asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a + b), "r"(n) : "memory");
        }
    }
    uint64_t t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    for (;;) {
        uint64_t t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        if (t - t0 >= ns) break;
    }
}
__global__ void empty_k(uint32_t* out) {
    if (threadIdx.x == 1234) out[0] = 1;
}

int main() {
    const uint64_t SB = 67108864ull;
    const uint64_t KVB = 4ull << 30;
    uint8_t *codes, *kv, *flush;
    uint32_t *o, *d_rows, *d_rows512;
    cudaMalloc(&codes, SB);
    cudaMalloc(&kv, KVB);
    cudaMalloc(&flush, 512ull << 20);
    cudaMalloc(&o, 4);
    cudaMemset(codes, 1, SB);
    cudaMemset(kv, 1, KVB);
    const uint32_t kk = 2622, P = 32;
    // 256-byte rows: K cache [32][131072][256 B] then V cache, same ids
    std::vector<uint32_t> rows(kk * 2 * P), rows512(kk * P);
    std::mt19937 g(3);
    const uint32_t n_tok = 131072;
    for (uint32_t p = 0; p < P; ++p) {
        std::vector<uint32_t> r(kk);
        for (auto& x : r) x = g() % n_tok;
        std::sort(r.begin(), r.end());
        for (uint32_t i = 0; i < kk; ++i) {
            rows[p * kk + i] = p * n_tok + r[i];                       // K
            rows[(P + p) * kk + i] = (P + p) * n_tok + r[i];           // V
            rows512[p * kk + i] = p * n_tok + r[i];                    // K|V token
        }
    }
    cudaMalloc(&d_rows, rows.size() * 4);
    cudaMalloc(&d_rows512, rows512.size() * 4);
    cudaMemcpy(d_rows, rows.data(), rows.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(d_rows512, rows512.data(), rows512.size() * 4, cudaMemcpyHostToDevice);
    cudaStream_t s;
    cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    auto flush_l2 = [&]() {
        cudaMemsetAsync(flush, 7, 512ull << 20, s);
        stream_chunk<<<444, 256, 0, s>>>(flush, (256ull << 20) / 32, o);
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
    auto run = [&](const char* name, std::function<void()> fn, double bytes) {
        const double t = graph_us([&] { flush_l2(); fn(); }) - base;
        printf("%-60s %8.2f us  %7.1f GB/s  %s\n", name, t, bytes / t / 1e3,
               cudaGetErrorString(cudaGetLastError()));
    };
    run("empty kernel", [&] { empty_k<<<1, 32, 0, s>>>(o); }, 0);
    run("stream 67MB", [&] { stream_chunk<<<444, 256, 0, s>>>(codes, SB / 32, o); }, SB);
    const double gb = (double)kk * 2 * P * 256;
    run("gather 43MB, 256B rows, warp x 8 rows", [&] { g_warp<256, 8><<<(kk * 2 * P / 8 * 32 + 127) / 128, 128, 0, s>>>(kv, d_rows, kk * 2 * P, o); }, gb);
    run("gather 43MB, 256B rows, warp x 4 rows", [&] { g_warp<256, 4><<<(kk * 2 * P / 4 * 32 + 127) / 128, 128, 0, s>>>(kv, d_rows, kk * 2 * P, o); }, gb);
    run("gather 43MB, 512B rows (K|V), warp x 4 rows", [&] { g_warp<512, 4><<<(kk * P / 4 * 32 + 127) / 128, 128, 0, s>>>(kv, d_rows512, kk * P, o); }, gb);
    run("gather 43MB, 512B rows (K|V), warp x 8 rows", [&] { g_warp<512, 8><<<(kk * P / 8 * 32 + 127) / 128, 128, 0, s>>>(kv, d_rows512, kk * P, o); }, gb);
    for (uint32_t us : {7u, 20u}) {
        const char* kinds[] = {"", "bulk prefetch", "line prefetch", "ldcg lines"};
        for (int pf = 1; pf <= 2; ++pf) {
            char nm[128];
            snprintf(nm, sizeof nm, "spin %u us (444 CTAs, stream's chunks) + %s, then stream", us, kinds[pf]);
            run(nm, [&] { spin_pf<<<444, 256, 0, s>>>(codes, SB, us * 1000, pf); stream_chunk<<<444, 256, 0, s>>>(codes, SB / 32, o); }, SB);
        }
    }
    for (uint32_t us : {7u, 20u}) {
        char nm[128];
        snprintf(nm, sizeof nm, "spin %u us (256 CTAs) then stream 67MB", us);
        run(nm, [&] { spin_pf<<<256, 128, 0, s>>>(codes, SB, us * 1000, 0); stream_chunk<<<444, 256, 0, s>>>(codes, SB / 32, o); }, SB);
        const char* kinds[] = {"", "bulk prefetch", "line prefetch", "ldcg lines"};
        for (int pf = 1; pf <= 3; ++pf) {
            snprintf(nm, sizeof nm, "spin %u us + %s 67MB, then stream 67MB", us, kinds[pf]);
            run(nm, [&] { spin_pf<<<256, 128, 0, s>>>(codes, SB, us * 1000, pf); stream_chunk<<<444, 256, 0, s>>>(codes, SB / 32, o); }, SB);
        }
    }
    run("stream 67MB, self bulk prefetch of each chunk", [&] { stream_chunk<<<444, 256, 0, s>>>(codes, SB / 32, o, 1); }, SB);
    run("stream 67MB twice (second L2-warm)", [&] { stream_chunk<<<444, 256, 0, s>>>(codes, SB / 32, o); stream_chunk<<<444, 256, 0, s>>>(codes, SB / 32, o); }, SB);
    run("stream 67MB then gather 43MB", [&] {
        stream_chunk<<<444, 256, 0, s>>>(codes, SB / 32, o);
        g_warp<256, 8><<<(kk * 2 * P / 8 * 32 + 127) / 128, 128, 0, s>>>(kv, d_rows, kk * 2 * P, o);
    }, SB + gb);
    return 0;
}
