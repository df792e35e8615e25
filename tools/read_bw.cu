// Microbenchmark (not part of the product): read-only HBM streaming ceiling
// on this B200 for the access patterns K3 can use. Reads a 268 MB buffer
// (the config-3 code cache) and XOR-reduces it.
//   A<U>: LDG.E.NA.EFL2.256, U units of 32 B in flight per thread, grid-stride
//   T<S>: cp.async.bulk (TMA 1-D) ring of S stages x 16 KB per CTA, consumer
//         warps XOR the staged data from shared memory
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o read_bw read_bw.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ void ld256(const uint32_t* p, uint32_t* w) {
    asm volatile("ld.global.nc.L1::no_allocate.L2::evict_first.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3]), "=r"(w[4]), "=r"(w[5]), "=r"(w[6]), "=r"(w[7])
                 : "l"(p));
}

template <int U>
__global__ void __launch_bounds__(256) rd_ldg(const uint32_t* __restrict__ a, uint64_t units, uint32_t* out) {
    uint32_t acc = 0;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (; i + (U - 1) * stride < units; i += U * stride) {
        uint32_t w[U][8];
#pragma unroll
        for (int u = 0; u < U; ++u) ld256(a + (i + u * stride) * 8, w[u]);
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
            for (int k = 0; k < 8; ++k) acc ^= w[u][k];
    }
    for (; i < units; i += stride) {
        uint32_t w[8];
        ld256(a + i * 8, w);
        for (int k = 0; k < 8; ++k) acc ^= w[k];
    }
    if (acc == 0x12345678u) out[0] = acc;
}

// contiguous-chunk variant (each CTA owns one range, like K3's segments)
template <int U>
__global__ void __launch_bounds__(256) rd_ldg_chunk(const uint32_t* __restrict__ a, uint64_t units, uint32_t* out) {
    const uint64_t per = (units + gridDim.x - 1) / gridDim.x;
    const uint64_t u0 = blockIdx.x * per, u1 = min(units, u0 + per);
    uint32_t acc = 0;
    for (uint64_t base = u0; base < u1; base += (uint64_t)U * 256) {
        uint32_t w[U][8];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint64_t i = base + u * 256 + threadIdx.x;
            if (i < u1) ld256(a + i * 8, w[u]); else for (int k = 0; k < 8; ++k) w[u][k] = 0;
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
            for (int k = 0; k < 8; ++k) acc ^= w[u][k];
    }
    if (acc == 0x12345678u) out[0] = acc;
}

// contiguous chunks with NT threads per CTA and double-buffered U-unit batches
// (the K3-fused stream loop shape)
template <int U, int NT>
__global__ void __launch_bounds__(NT) rd_chunk_db(const uint32_t* __restrict__ a, uint64_t units, uint32_t* out) {
    const uint64_t per = (units + gridDim.x - 1) / gridDim.x;
    const uint64_t u0 = blockIdx.x * per, u1 = min(units, u0 + per);
    uint32_t acc = 0;
    uint32_t wa[U][8], wb[U][8];
    auto load = [&](uint32_t (*w)[8], uint64_t base) {
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint64_t i = base + u * NT + threadIdx.x;
            if (i < u1) ld256(a + i * 8, w[u]); else for (int k = 0; k < 8; ++k) w[u][k] = 0;
        }
    };
    auto use = [&](uint32_t (*w)[8]) {
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
            for (int k = 0; k < 8; ++k) acc += __popc(w[u][k]);
    };
    const uint64_t step = (uint64_t)U * NT;
    load(wa, u0);
    for (uint64_t base = u0; base < u1; base += 2 * step) {
        if (base + step < u1) load(wb, base + step);
        use(wa);
        if (base + step < u1) {
            if (base + 2 * step < u1) load(wa, base + 2 * step);
            use(wb);
        }
    }
    if (acc == 0x12345678u) out[0] = acc;
}

// single-buffered chunk loop, NT threads, optional popcount use
template <int U, int NT, bool POPC>
__global__ void __launch_bounds__(NT) rd_chunk_sb(const uint32_t* __restrict__ a, uint64_t units, uint32_t* out) {
    const uint64_t per = (units + gridDim.x - 1) / gridDim.x;
    const uint64_t u0 = blockIdx.x * per, u1 = min(units, u0 + per);
    uint32_t acc = 0;
    for (uint64_t base = u0; base < u1; base += (uint64_t)U * NT) {
        uint32_t w[U][8];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint64_t i = base + u * NT + threadIdx.x;
            if (i < u1) ld256(a + i * 8, w[u]); else for (int k = 0; k < 8; ++k) w[u][k] = 0;
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
            for (int k = 0; k < 8; ++k) acc = POPC ? acc + __popc(w[u][k]) : acc ^ w[u][k];
    }
    if (acc == 0x12345678u) out[0] = acc;
}

// chunk read + one u16 score write per 32-byte unit (K3 two-pass shape):
// scores go to a global array that stays L2-resident (16.7 MB)
template <int U>
__global__ void __launch_bounds__(256) rd_chunk_wr(const uint32_t* __restrict__ a, uint64_t units, uint16_t* sc) {
    const uint64_t per = (units + gridDim.x - 1) / gridDim.x;
    const uint64_t u0 = blockIdx.x * per, u1 = min(units, u0 + per);
    for (uint64_t base = u0; base < u1; base += (uint64_t)U * 256) {
        uint32_t w[U][8];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint64_t i = base + u * 256 + threadIdx.x;
            if (i < u1) ld256(a + i * 8, w[u]); else for (int k = 0; k < 8; ++k) w[u][k] = 0;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint64_t i = base + u * 256 + threadIdx.x;
            uint32_t m0 = 0, m1 = 0;
#pragma unroll
            for (int k = 0; k < 4; ++k) { m0 += __popc(w[u][k]); m1 += __popc(w[u][k + 4]); }
            if (i < u1) sc[i] = (uint16_t)(m0 | (m1 << 8));
        }
    }
}

// K3-fused-v2 pattern: CPP CTAs per problem, tiles of 256 units dealt
// round-robin, KB tiles per load batch, double buffered
template <int KB>
__global__ void __launch_bounds__(256) rd_tiles(const uint32_t* __restrict__ a, uint32_t P, uint32_t CPP,
                                                uint32_t units_per_p, uint32_t* out) {
    const uint32_t p = blockIdx.x / CPP, c = blockIdx.x % CPP;
    const uint32_t ntiles = units_per_p / 256;
    const uint32_t mt = ntiles > c ? (ntiles - c + CPP - 1) / CPP : 0;
    const uint32_t* base = a + (uint64_t)p * units_per_p * 8;
    uint32_t acc = 0;
    for (uint32_t t0 = 0; t0 < mt; t0 += KB) {
        uint32_t w[KB][8];
#pragma unroll
        for (int i = 0; i < KB; ++i)
            if (t0 + i < mt) ld256(base + ((uint64_t)(c + (t0 + i) * CPP) * 256 + threadIdx.x) * 8, w[i]);
            else for (int k = 0; k < 8; ++k) w[i][k] = 0;
#pragma unroll
        for (int i = 0; i < KB; ++i)
#pragma unroll
            for (int k = 0; k < 8; ++k) acc ^= w[i][k];
    }
    if (acc == 0x12345678u) out[0] = acc;
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int S, uint32_t CH = 16384>
__global__ void __launch_bounds__(512) rd_tma(const uint8_t* __restrict__ a, uint64_t bytes, uint32_t* out) {
    extern __shared__ __align__(128) uint8_t sm[];
    __shared__ __align__(8) uint64_t full[S], empty[S];
    const uint64_t nch = bytes / CH;
    const uint64_t per = (nch + gridDim.x - 1) / gridDim.x;
    const uint64_t c0 = blockIdx.x * per, c1 = min(nch, c0 + per);
    const int tid = threadIdx.x;
    if (tid == 0) {
        for (int s = 0; s < S; ++s) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(smem_u32(&full[s])));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(smem_u32(&empty[s])), "r"(blockDim.x));
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    auto issue = [&](uint64_t c) {
        const int s = (int)((c - c0) % S);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(smem_u32(&full[s])), "r"(CH) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     :: "r"(smem_u32(sm + s * CH)), "l"(a + c * CH), "r"(CH), "r"(smem_u32(&full[s])) : "memory");
    };
    if (tid == 0)
        for (uint64_t c = c0; c < min(c1, c0 + S); ++c) issue(c);
    uint32_t acc = 0;
    for (uint64_t c = c0; c < c1; ++c) {
        const int s = (int)((c - c0) % S);
        const uint32_t ph = (uint32_t)(((c - c0) / S) & 1);
        uint32_t done = 0;
        while (!done)
            asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p; }"
                         : "=r"(done) : "r"(smem_u32(&full[s])), "r"(ph) : "memory");
        const uint4* v = reinterpret_cast<const uint4*>(sm + s * CH);
#pragma unroll
        for (uint32_t k = tid; k < CH / 16; k += blockDim.x) {
            const uint4 x = v[k];
            acc ^= x.x ^ x.y ^ x.z ^ x.w;
        }
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"(smem_u32(&empty[s])) : "memory");
        if (tid == 0 && c + S < c1) {
            done = 0;
            while (!done)
                asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p; }"
                             : "=r"(done) : "r"(smem_u32(&empty[s])), "r"(ph) : "memory");
            issue(c + S);
        }
    }
    if (acc == 0x12345678u) out[0] = acc;
}

int main() {
    const uint64_t bytes = 268435456ull;
    uint32_t* a; uint32_t* o;
    cudaMalloc(&a, bytes); cudaMalloc(&o, 4);
    uint32_t* a2; cudaMalloc(&a2, bytes / 16);
    cudaMemset(a, 1, bytes);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    auto timeit = [&](const char* name, auto launch) {
        for (int i = 0; i < 3; ++i) launch();
        cudaEventRecord(e0);
        for (int i = 0; i < 20; ++i) launch();
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1); ms /= 20;
        cudaError_t err = cudaGetLastError();
        printf("%-28s %8.2f us  %7.1f GB/s  %s\n", name, ms * 1000, bytes / (ms * 1e-3) / 1e9, err ? cudaGetErrorString(err) : "");
    };
    const uint64_t units = bytes / 32;
    for (int occ : {2, 3, 4, 8}) {
        char n[64];
        snprintf(n, 64, "ldg256 U2 grid=%dx", occ); timeit(n, [&] { rd_ldg<2><<<sms * occ, 256>>>(a, units, o); });
        snprintf(n, 64, "ldg256 U4 grid=%dx", occ); timeit(n, [&] { rd_ldg<4><<<sms * occ, 256>>>(a, units, o); });
        snprintf(n, 64, "ldg256 U8 grid=%dx", occ); timeit(n, [&] { rd_ldg<8><<<sms * occ, 256>>>(a, units, o); });
        snprintf(n, 64, "chunk U4 grid=%dx", occ); timeit(n, [&] { rd_ldg_chunk<4><<<sms * occ, 256>>>(a, units, o); });
        snprintf(n, 64, "chunk U8 grid=%dx", occ); timeit(n, [&] { rd_ldg_chunk<8><<<sms * occ, 256>>>(a, units, o); });
    }
    {
        // same patterns with K3-fused's shared-memory carve-out (72 KB/CTA,
        // 3 CTAs/SM): does the tiny L1 left over throttle the loads?
        const int pad = 72 * 1024;
        cudaFuncSetAttribute(rd_ldg_chunk<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, pad);
        cudaFuncSetAttribute(rd_ldg_chunk<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, pad);
        cudaFuncSetAttribute(rd_ldg<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, pad);
        cudaFuncSetAttribute(rd_ldg<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, pad);
        timeit("chunk U2 3x smem72K", [&] { rd_ldg_chunk<2><<<sms * 3, 256, pad>>>(a, units, o); });
        timeit("chunk U4 3x smem72K", [&] { rd_ldg_chunk<4><<<sms * 3, 256, pad>>>(a, units, o); });
        timeit("ldg256 U2 3x smem72K", [&] { rd_ldg<2><<<sms * 3, 256, pad>>>(a, units, o); });
        timeit("ldg256 U4 3x smem72K", [&] { rd_ldg<4><<<sms * 3, 256, pad>>>(a, units, o); });
        for (int kb : {20, 24, 28, 30, 32, 33, 36, 40, 44, 52, 56, 60, 64, 68, 70, 72}) {
            const int pd = kb * 1024;
            char n[64];
            cudaFuncSetAttribute(rd_ldg_chunk<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, pd);
            int occ = 0;
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, rd_ldg_chunk<2>, 256, pd);
            snprintf(n, 64, "sweep chunk U2 3x smem%dK occ%d", kb, occ); timeit(n, [&] { rd_ldg_chunk<2><<<sms * 3, 256, pd>>>(a, units, o); });
        }
        {
            auto run = [&](const char* name, auto k, int grid, int nt, int kb) {
                cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, kb * 1024);
                int occ = 0;
                cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, nt, kb * 1024);
                char n[80];
                snprintf(n, 80, "%s g%d smem%dK occ%d", name, grid, kb, occ);
                timeit(n, [&] { k<<<grid, nt, kb * 1024>>>(a, units, o); });
            };
            run("db U4 NT128", rd_chunk_db<4, 128>, 576, 128, 47);
            run("db U4 NT128", rd_chunk_db<4, 128>, 592, 128, 47);
            run("db U2 NT128", rd_chunk_db<2, 128>, 576, 128, 47);
            run("db U2 NT256", rd_chunk_db<2, 256>, 444, 256, 60);
            run("db U1 NT256", rd_chunk_db<1, 256>, 444, 256, 60);
            run("db U4 NT128", rd_chunk_db<4, 128>, 576, 128, 0);
            run("db U2 NT256", rd_chunk_db<2, 256>, 444, 256, 0);
            run("db U8 NT128", rd_chunk_db<8, 128>, 576, 128, 47);
            run("sb U4 NT128 xor", rd_chunk_sb<4, 128, false>, 576, 128, 47);
            run("sb U4 NT128 popc", rd_chunk_sb<4, 128, true>, 576, 128, 47);
            run("sb U8 NT128 popc", rd_chunk_sb<8, 128, true>, 576, 128, 47);
            run("sb U2 NT256 xor", rd_chunk_sb<2, 256, false>, 444, 256, 60);
            run("sb U2 NT256 popc", rd_chunk_sb<2, 256, true>, 444, 256, 60);
            run("sb U4 NT256 popc", rd_chunk_sb<4, 256, true>, 444, 256, 60);
            run("sb U4 NT128 popc", rd_chunk_sb<4, 128, true>, 592, 128, 47);
            run("sb U6 NT128 popc", rd_chunk_sb<6, 128, true>, 576, 128, 47);
        }
        for (int co : {50, 75, 100}) {
            const int pd = 33 * 1024;
            char n[64];
            cudaFuncSetAttribute(rd_ldg_chunk<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, pd);
            cudaFuncSetAttribute(rd_ldg_chunk<2>, cudaFuncAttributePreferredSharedMemoryCarveout, co);
            snprintf(n, 64, "sweep chunk U2 3x smem33K carve%d", co); timeit(n, [&] { rd_ldg_chunk<2><<<sms * 3, 256, pd>>>(a, units, o); });
        }
        cudaFuncSetAttribute(rd_ldg_chunk<2>, cudaFuncAttributePreferredSharedMemoryCarveout, -1);
        for (int kb : {0, 16, 33, 48}) {
            const int pd = kb * 1024;
            char n[64];
            cudaFuncSetAttribute(rd_ldg_chunk<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, pd);
            cudaFuncSetAttribute(rd_chunk_wr<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, pd);
            cudaFuncSetAttribute(rd_chunk_wr<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, pd);
            snprintf(n, 64, "chunk U2 3x smem%dK", kb); timeit(n, [&] { rd_ldg_chunk<2><<<sms * 3, 256, pd>>>(a, units, o); });
            snprintf(n, 64, "chunk+wr U2 3x smem%dK", kb); timeit(n, [&] { rd_chunk_wr<2><<<sms * 3, 256, pd>>>(a, units, (uint16_t*)(a2)); });
            snprintf(n, 64, "chunk+wr U4 2x smem%dK", kb); timeit(n, [&] { rd_chunk_wr<4><<<sms * 2, 256, pd>>>(a, units, (uint16_t*)(a2)); });
        }
        timeit("chunk U2 443 smem72K", [&] { rd_ldg_chunk<2><<<443, 256, pad>>>(a, units, o); });
        timeit("chunk U2 3x", [&] { rd_ldg_chunk<2><<<sms * 3, 256>>>(a, units, o); });
    }
    {
        const uint32_t upp = (uint32_t)(units / 32);
        timeit("tiles KB4 CPP9 (288)", [&] { rd_tiles<4><<<32 * 9, 256>>>(a, 32, 9, upp, o); });
        timeit("tiles KB8 CPP9 (288)", [&] { rd_tiles<8><<<32 * 9, 256>>>(a, 32, 9, upp, o); });
        timeit("tiles KB4 CPP13 (416)", [&] { rd_tiles<4><<<32 * 13, 256>>>(a, 32, 13, upp, o); });
        timeit("tiles KB2 CPP13 (416)", [&] { rd_tiles<2><<<32 * 13, 256>>>(a, 32, 13, upp, o); });
        for (int kb : {0, 58}) {
            cudaFuncSetAttribute(rd_tiles<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, kb * 1024);
            cudaFuncSetAttribute(rd_tiles<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, kb * 1024);
            char n[64];
            snprintf(n, 64, "tiles KB2 CPP13 (416) smem%dK", kb);
            timeit(n, [&] { rd_tiles<2><<<32 * 13, 256, kb * 1024>>>(a, 32, 13, upp, o); });
            snprintf(n, 64, "tiles KB4 CPP13 (416) smem%dK", kb);
            timeit(n, [&] { rd_tiles<4><<<32 * 13, 256, kb * 1024>>>(a, 32, 13, upp, o); });
            cudaFuncSetAttribute(rd_ldg_chunk<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, kb * 1024);
            snprintf(n, 64, "chunk U2 grid=416 smem%dK", kb);
            timeit(n, [&] { rd_ldg_chunk<2><<<416, 256, kb * 1024>>>(a, units, o); });
            cudaFuncSetAttribute(rd_ldg<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, kb * 1024);
            snprintf(n, 64, "ldg256 U2 grid=416 smem%dK", kb);
            timeit(n, [&] { rd_ldg<2><<<416, 256, kb * 1024>>>(a, units, o); });
        }
        timeit("chunk U4 grid=288", [&] { rd_ldg_chunk<4><<<288, 256>>>(a, units, o); });
        timeit("ldg256 U4 grid=288", [&] { rd_ldg<4><<<288, 256>>>(a, units, o); });
    }
    {
        // TMA ring at the fused kernel's budget: 1 CTA/SM, 512 threads,
        // ~176 KB of the CTA's shared memory taken by counters + scores
        auto run = [&](const char* name, auto k, int ring, int thr) {
            const int dyn = ring + 176 * 1024;
            cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn);
            timeit(name, [&] { k<<<sms, thr, dyn>>>((const uint8_t*)a, bytes, o); });
        };
        run("tma S3x16K 1x512 +176K", rd_tma<3, 16384>, 3 * 16384, 512);
        run("tma S4x12K 1x512 +176K", rd_tma<4, 12288>, 4 * 12288, 512);
        run("tma S6x8K 1x512 +176K", rd_tma<6, 8192>, 6 * 8192, 512);
        run("tma S3x16K 1x256 +176K", rd_tma<3, 16384>, 3 * 16384, 256);
        run("tma S2x16K 1x512 +176K", rd_tma<2, 16384>, 2 * 16384, 512);
    }
    for (int occ : {1, 2}) {
        char n[64];
        cudaFuncSetAttribute(rd_tma<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * 16384);
        cudaFuncSetAttribute(rd_tma<6>, cudaFuncAttributeMaxDynamicSharedMemorySize, 6 * 16384);
        cudaFuncSetAttribute(rd_tma<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * 16384);
        snprintf(n, 64, "tma S4 grid=%dx", occ); timeit(n, [&] { rd_tma<4><<<sms * occ, 256, 4 * 16384>>>((const uint8_t*)a, bytes, o); });
        snprintf(n, 64, "tma S6 grid=%dx", occ); timeit(n, [&] { rd_tma<6><<<sms * occ, 256, 6 * 16384>>>((const uint8_t*)a, bytes, o); });
        if (occ == 1) { snprintf(n, 64, "tma S8 grid=%dx", occ); timeit(n, [&] { rd_tma<8><<<sms * occ, 256, 8 * 16384>>>((const uint8_t*)a, bytes, o); }); }
    }
    return 0;
}
