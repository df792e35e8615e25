// Probe (not part of the product): TMEM -> register read throughput of one
// SM (tcgen05.ld.sync.aligned.32x32b.x32 sweeps over 512 columns by W warps,
// W/4 warps per lane quarter), the bound on K2's epilogues.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tmem_read_bw tmem_read_bw.cu
#include <cstdio>
#include <cstdint>

__global__ void probe(int reps, long long* out, uint32_t* sink) {
    __shared__ uint32_t s_tmem;
    const int warp = threadIdx.x >> 5;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;"
                     :: "r"((uint32_t)__cvta_generic_to_shared(&s_tmem)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t base = s_tmem;
    const uint32_t quarter = warp & 3, nw = blockDim.x / 32, group = warp / 4, ngroups = nw / 4;
    uint32_t acc = 0;
    __syncthreads();
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
        for (uint32_t c = group * 32; c < 512; c += ngroups * 32) {
            uint32_t v[32];
            const uint32_t addr = base + ((quarter * 32) << 16) + c;
            asm volatile(
                "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
                "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                  "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
                  "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
                  "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
                : "r"(addr));
            asm volatile("tcgen05.wait::ld.sync.aligned;");
#pragma unroll
            for (int i = 0; i < 32; ++i) acc ^= v[i];
        }
    }
    __syncthreads();
    long long t1 = clock64();
    if (threadIdx.x == 0) out[0] = t1 - t0;
    if (acc == 0x12345u) sink[0] = acc;
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" :: "r"(base));
}

int main() {
    long long* o; uint32_t* s;
    cudaMallocManaged(&o, 8); cudaMalloc(&s, 4);
    const int reps = 200;
    for (int w : {4, 8, 16}) {
        probe<<<1, w * 32>>>(reps, o, s);
        cudaError_t e = cudaDeviceSynchronize();
        const double bytes = (double)reps * 512 * 128 * 4;  // every column of every lane, reps times
        printf("warps %2d: %lld cycles, %.1f B/clk/SM  %s\n", w, o[0], bytes / o[0], cudaGetErrorString(e));
    }
    return 0;
}
