// Throughput microbenchmarks (not product code): IDP4A, IMMA mma.sync m16n8k32 u8, IMAD.WIDE.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ubench tools/ubench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void k_dp4a(uint32_t* out, int iters) {
    uint32_t a[8], acc[8];
    for (int i = 0; i < 8; ++i) { a[i] = threadIdx.x * (i + 1); acc[i] = i; }
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int i = 0; i < 8; ++i) acc[i] = __dp4a(a[i], a[(i + 1) & 7], acc[i]);
    uint32_t s = 0;
    for (int i = 0; i < 8; ++i) s += acc[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_imma(uint32_t* out, int iters) {
    uint32_t a[4], b[2];
    int c[4][4] = {};
    for (int i = 0; i < 4; ++i) a[i] = threadIdx.x * (i + 3);
    b[0] = threadIdx.x; b[1] = threadIdx.x * 7;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int j = 0; j < 4; ++j)
            asm volatile("mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                         : "+r"(c[j][0]), "+r"(c[j][1]), "+r"(c[j][2]), "+r"(c[j][3])
                         : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
    }
    int s = 0;
    for (int j = 0; j < 4; ++j) for (int i = 0; i < 4; ++i) s += c[j][i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_imadwide(uint32_t* out, int iters, int a0, int b0) {
    long long acc[4] = {0, 1, 2, 3};
    int x = threadIdx.x, y = threadIdx.x * 3;
    uint32_t cnt = 0;
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            long long v = (long long)(a0 + j) * (x + it) + (long long)(b0 - j) * (y - it) - acc[j];
            cnt += v >= 0;
        }
    out[blockIdx.x * blockDim.x + threadIdx.x] = cnt;
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    uint32_t* out;
    cudaMalloc(&out, 1 << 26);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    int blocks = sms * 8, threads = 256, iters = 4096;
    float ms;
    for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(e0);
        k_dp4a<<<blocks, threads>>>(out, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        double dp4a = (double)blocks * threads * iters * 8;
        printf("dp4a: %.1f G dp4a/s = %.1f TMAC/s int8\n", dp4a / ms / 1e6, 4 * dp4a / ms / 1e9);
        cudaEventRecord(e0);
        k_imma<<<blocks, threads>>>(out, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        double mma = (double)blocks * (threads / 32) * iters * 4;
        printf("imma m16n8k32: %.1f T mma/s = %.1f TMAC/s int8\n", mma / ms / 1e9, mma * 4096 / ms / 1e9);
        cudaEventRecord(e0);
        k_imadwide<<<blocks, threads>>>(out, iters, 12345, -777);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        double t = (double)blocks * threads * iters * 4;
        printf("heaviside test (2 imad.wide): %.1f G tests/s\n", t / ms / 1e6);
    }
    int clk;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    printf("sms %d clock %d kHz\n", sms, clk);
    return 0;
}
