// Microbenchmark: latency of a GPU-scope all-to-all progress exchange (one counter per round,
// red.release.gpu add by one thread per CTA, ld.acquire.gpu polling), the cross-cluster handoff a
// multi-cluster decision kernel would need per colour class.  nvcc -gencode arch=compute_100a,code=sm_100a
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_rounds(unsigned int* cnt, int rounds, int payload_words, unsigned int* data) {
    const unsigned int n = gridDim.x;
    for (int r = 0; r < rounds; ++r) {
        if (threadIdx.x < payload_words) data[(r & 63) * 1024 + blockIdx.x * payload_words + threadIdx.x] = r;
        __syncthreads();
        if (threadIdx.x == 0) {
            asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(cnt + r) : "memory");
            unsigned int v;
            do {
                asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(cnt + r) : "memory");
            } while (v < n);
        }
        __syncthreads();
        if (threadIdx.x < 32) {  // read everybody's payload
            unsigned int s = 0;
            for (unsigned int j = threadIdx.x; j < n * payload_words; j += 32) s += data[(r & 63) * 1024 + j];
            if (s == 0xffffffff) data[0] = s;
        }
    }
}
int main() {
    const int rounds = 4096;
    unsigned int *cnt, *data;
    cudaMalloc(&cnt, rounds * 4);
    cudaMalloc(&data, 64 * 1024 * 4 * 4);
    for (int n : {16, 32, 64, 128, 148}) for (int pw : {0, 4}) {
        cudaMemset(cnt, 0, rounds * 4);
        cudaEvent_t a, b;
        cudaEventCreate(&a); cudaEventCreate(&b);
        k_rounds<<<n, 256>>>(cnt, 64, pw, data);
        cudaMemset(cnt, 0, rounds * 4);
        cudaEventRecord(a);
        k_rounds<<<n, 256>>>(cnt, rounds, pw, data);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        printf("ctas %3d payload %d words: %.3f us per round (%s)\n", n, pw, ms * 1e3 / rounds, cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
