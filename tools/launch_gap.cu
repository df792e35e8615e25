// Back-to-back launch floor for K3-fused's grid shape (not part of the product):
// 416 CTAs x 256 threads, 57 KB dynamic smem, plain vs cooperative launch, in
// a stream and captured in a CUDA graph. Prints us per launch.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o build/launch_gap tools/launch_gap.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(256, 3) empty_k(uint32_t* out, int touch) {
    extern __shared__ uint8_t sm[];
    if (touch) {  // zero 16 KB of smem like the K3 prologue
        for (int i = threadIdx.x; i < 4096; i += 256) reinterpret_cast<uint32_t*>(sm)[i] = 0;
        __syncthreads();
        if (sm[threadIdx.x] == 7) out[0] = 1;
    }
}

int main() {
    uint32_t* o;
    cudaMalloc(&o, 4);
    const int smem = 57 * 1024, G = 416;
    cudaFuncSetAttribute(empty_k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaStream_t s;
    cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int N = 200;
    for (int touch = 0; touch < 2; ++touch)
        for (int coop = 0; coop < 2; ++coop) {
            auto launch = [&] {
                void* args[] = {&o, &touch};
                if (coop)
                    cudaLaunchCooperativeKernel((const void*)empty_k, dim3(G), dim3(256), args, smem, s);
                else
                    cudaLaunchKernel((const void*)empty_k, dim3(G), dim3(256), args, smem, s);
            };
            for (int i = 0; i < 10; ++i) launch();
            cudaEventRecord(a, s);
            for (int i = 0; i < N; ++i) launch();
            cudaEventRecord(b, s);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            // graph of one launch, replayed
            cudaGraph_t g;
            cudaGraphExec_t ge;
            cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
            launch();
            cudaStreamEndCapture(s, &g);
            cudaGraphInstantiate(&ge, g, 0);
            for (int i = 0; i < 10; ++i) cudaGraphLaunch(ge, s);
            cudaEventRecord(a, s);
            for (int i = 0; i < N; ++i) cudaGraphLaunch(ge, s);
            cudaEventRecord(b, s);
            cudaEventSynchronize(b);
            float ms2;
            cudaEventElapsedTime(&ms2, a, b);
            printf("touch=%d coop=%d  stream %.2f us/launch  graph %.2f us/launch  %s\n", touch, coop,
                   ms * 1e3 / N, ms2 * 1e3 / N, cudaGetErrorString(cudaGetLastError()));
            cudaGraphExecDestroy(ge);
            cudaGraphDestroy(g);
        }
    return 0;
}
