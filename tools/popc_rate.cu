// POPC / LOP3 / IADD issue-rate microbenchmark (sm_100a).
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o build/popc_rate tools/popc_rate.cu
// Prints warp-instructions per cycle per SM for each op, so the K3 inner
// loop's pipe budget (8 POPC + ~20 ALU per 32-byte unit) can be checked.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int OP>
__global__ void __launch_bounds__(256) spin(uint32_t seed, int iters, uint32_t* out) {
    uint32_t x[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = seed * (threadIdx.x + 1) + i * 0x9e3779b9u;
    uint32_t acc = 0;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            if (OP == 0) {
                acc += __popc(x[i]);  // POPC + IADD
                x[i] = x[i] * 3u;     // keep inputs changing (IMAD)
            } else if (OP == 1) {
                x[i] = (x[i] ^ acc) & (x[(i + 1) & 7] | 0x55u);  // LOP3
                acc ^= x[i];
            } else {
                acc += x[i];  // IADD only
                x[i] = x[i] * 3u;
            }
        }
    }
    if (acc == 0x12345678u) out[0] = acc;
}

int main() {
    int sms = 0, clk = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);  // kHz
    uint32_t* o;
    cudaMalloc(&o, 4);
    const int iters = 4096, blocks = sms * 4;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    auto run = [&](const char* name, auto k, int ops_per_iter) {
        k<<<blocks, 256>>>(1u, iters, o);
        cudaEventRecord(a);
        k<<<blocks, 256>>>(1u, iters, o);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms = 0;
        cudaEventElapsedTime(&ms, a, b);
        const double warp_ops = (double)blocks * 8 * iters * ops_per_iter;
        const double cyc = ms * 1e-3 * clk * 1e3;
        printf("%-28s %.3f ms  %.2f warp-op/clk/SM (target op)\n", name, ms, warp_ops / cyc / sms);
    };
    run("POPC(+IADD+IMAD) x8", spin<0>, 8);
    run("LOP3-chain x8", spin<1>, 8);
    run("IADD(+IMAD) x8", spin<2>, 8);
    printf("clock %d MHz, %d SMs\n", clk / 1000, sms);
    return 0;
}
