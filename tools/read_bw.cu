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

template <int S>
__global__ void __launch_bounds__(256) rd_tma(const uint8_t* __restrict__ a, uint64_t bytes, uint32_t* out) {
    constexpr uint32_t CH = 16384;
    extern __shared__ __align__(128) uint8_t sm[];
    __shared__ __align__(8) uint64_t full[S], empty[S];
    const uint64_t nch = bytes / CH;
    const uint64_t per = (nch + gridDim.x - 1) / gridDim.x;
    const uint64_t c0 = blockIdx.x * per, c1 = min(nch, c0 + per);
    const int tid = threadIdx.x;
    if (tid == 0) {
        for (int s = 0; s < S; ++s) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(smem_u32(&full[s])));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 256;" :: "r"(smem_u32(&empty[s])));
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
        for (int k = 0; k < (int)(CH / 16 / 256); ++k) {
            const uint4 x = v[k * 256 + tid];
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
        const uint32_t upp = (uint32_t)(units / 32);
        timeit("tiles KB4 CPP9 (288)", [&] { rd_tiles<4><<<32 * 9, 256>>>(a, 32, 9, upp, o); });
        timeit("tiles KB8 CPP9 (288)", [&] { rd_tiles<8><<<32 * 9, 256>>>(a, 32, 9, upp, o); });
        timeit("tiles KB4 CPP13 (416)", [&] { rd_tiles<4><<<32 * 13, 256>>>(a, 32, 13, upp, o); });
        timeit("tiles KB2 CPP13 (416)", [&] { rd_tiles<2><<<32 * 13, 256>>>(a, 32, 13, upp, o); });
        timeit("chunk U4 grid=288", [&] { rd_ldg_chunk<4><<<288, 256>>>(a, units, o); });
        timeit("ldg256 U4 grid=288", [&] { rd_ldg<4><<<288, 256>>>(a, units, o); });
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
