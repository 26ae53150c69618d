// L2-resident read bandwidth (not product code): every SM streams a 48 MB buffer (fits the
// 126 MB L2) with 16-B loads, many times; reports GB/s after a warm-up pass.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void rd(const uint4* __restrict__ a, size_t n, int reps, unsigned long long* out) {
    uint4 acc = make_uint4(0, 0, 0, 0);
    for (int r = 0; r < reps; ++r)
        for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
            uint4 v = __ldcg(a + i);
            acc.x ^= v.x; acc.y ^= v.y; acc.z ^= v.z; acc.w ^= v.w;
        }
    if ((acc.x ^ acc.y ^ acc.z ^ acc.w) == 0x12345678u) out[0] = 1;
}
int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    for (size_t mb : {24, 48, 96, 2048}) {
        size_t bytes = mb << 20, n = bytes / 16;
        uint4* a; cudaMalloc(&a, bytes); cudaMemset(a, 1, bytes);
        unsigned long long* o; cudaMalloc(&o, 8);
        int reps = mb >= 1024 ? 2 : 20;
        rd<<<sms * 4, 512>>>(a, n, 1, o);
        cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
        cudaEventRecord(e0); rd<<<sms * 4, 512>>>(a, n, reps, o); cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        printf("buffer %5zu MB: %.1f GB/s\n", mb, (double)bytes * reps / ms / 1e6);
        cudaFree(a); cudaFree(o);
    }
}
