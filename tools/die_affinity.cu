// Does it matter WHICH SM streams which contiguous chunk? (not part of the
// product). 444 CTAs x 256 threads (3/SM), each reads one 604 KB chunk of a
// 268 MB buffer with LDG.256 (K3's stream shape). Chunk choice:
//   block  : chunk = blockIdx
//   ticket : chunk = arrival order (atomic ticket)
//   sm     : chunk = 3 * smid + slot     (SM s reads region s of 148)
//   sm_rev : chunk = 3 * ((smid + 74) % 148) + slot
//   sm_perm: chunk = 3 * perm(smid) + slot, perm = multiplicative scramble
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o build/die_affinity tools/die_affinity.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ void ld256(const uint32_t* p, uint32_t* w) {
    asm volatile("ld.global.nc.L1::no_allocate.L2::evict_first.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3]), "=r"(w[4]), "=r"(w[5]), "=r"(w[6]), "=r"(w[7])
                 : "l"(p));
}

__global__ void __launch_bounds__(256, 3) rd(const uint32_t* __restrict__ a, uint64_t units, int mode,
                                             uint32_t* ctr, uint32_t* out) {
    __shared__ uint32_t s_chunk;
    if (threadIdx.x == 0) {
        uint32_t smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        uint32_t c = blockIdx.x;
        if (mode == 1) c = atomicAdd(ctr, 1u);
        if (mode >= 2) {
            const uint32_t slot = atomicAdd(ctr + 1 + smid, 1u) % 3;
            uint32_t s = smid;
            if (mode == 3) s = (smid + 74) % 148;
            if (mode == 4) s = (smid * 37u + 11u) % 148;
            c = s * 3 + slot;
        }
        s_chunk = c;
    }
    __syncthreads();
    const uint32_t nch = gridDim.x;
    const uint64_t per = (units + nch - 1) / nch;
    const uint64_t u0 = (uint64_t)s_chunk * per, u1 = min(units, u0 + per);
    uint32_t acc = 0;
    for (uint64_t base = u0; base < u1; base += 2 * 256) {
        uint32_t w[2][8];
#pragma unroll
        for (int u = 0; u < 2; ++u) {
            const uint64_t i = base + u * 256 + threadIdx.x;
            if (i < u1) ld256(a + i * 8, w[u]); else for (int k = 0; k < 8; ++k) w[u][k] = 0;
        }
#pragma unroll
        for (int u = 0; u < 2; ++u)
#pragma unroll
            for (int k = 0; k < 8; ++k) acc += __popc(w[u][k]);
    }
    if (acc == 0x12345678u) out[0] = acc;
}

int main() {
    const uint64_t bytes = 268435456ull, units = bytes / 32;
    uint32_t *a, *o, *ctr;
    cudaMalloc(&a, bytes);
    cudaMalloc(&o, 4);
    cudaMalloc(&ctr, 4 * 256);
    cudaMemset(a, 1, bytes);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int smem = 57 * 1024;  // K3-fused's carve-out class (<= 196 KB/SM)
    cudaFuncSetAttribute(rd, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const char* names[] = {"block", "ticket", "sm", "sm_rev", "sm_perm"};
    for (int rep = 0; rep < 2; ++rep)
        for (int mode = 0; mode < 5; ++mode) {
            float tot = 0;
            for (int i = 0; i < 23; ++i) {
                cudaMemset(ctr, 0, 4 * 256);
                cudaEventRecord(e0);
                rd<<<sms * 3, 256, smem>>>(a, units, mode, ctr, o);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
                float ms;
                cudaEventElapsedTime(&ms, e0, e1);
                if (i >= 3) tot += ms;
            }
            tot /= 20;
            printf("%-8s %8.2f us  %7.1f GB/s  %s\n", names[mode], tot * 1e3, bytes / (tot * 1e-3) / 1e9,
                   cudaGetErrorString(cudaGetLastError()));
        }
    return 0;
}
