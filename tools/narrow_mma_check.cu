// Exactness / layout check of tcgen05.mma kind::f8f6f4 on TMA-unpacked narrow operands (not product
// code).  A [128][K] and B [N][K] hold small integers stored packed in global memory
// (e2m1: 16 x 4 bit in 8 bytes, CU_TENSOR_MAP_DATA_TYPE_16U4_ALIGN16B; e3m2: 16 x 6 bit in 12 bytes,
// 16U6_ALIGN16B), TMA-unpacked into the 128-B-swizzled K-major shared-memory layout, multiplied with
// fp32 accumulation in TMEM over K = 8192, and compared with the exact integer Gram on the host.
// Worst-case magnitudes: all |v| = 4 (e2m1) or 8 (e3m2), so the sum reaches K * 16 = 2^17 and
// K * 64 = 2^19 -- exact only if the tensor core accumulates with the full fp32 mantissa.
// mx = 1: the same e2m1 operands left PACKED (plain UINT8 TMA, 256 values per 128-B row) and
// multiplied with kind::mxf4.block_scale.block32 (K = 64 per instruction) with every ue8m0 scale
// factor = 2^0 (0x7F, written to TMEM columns [sfcol, sfcol + 8) by tcgen05.st), N = n columns.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/nmc tools/narrow_mma_check.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

constexpr int M = 128, N = 256, K = 8192;

__device__ __forceinline__ uint64_t sdesc(uint32_t saddr) {  // K-major, SWIZZLE_128B, SBO = 1024
    return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) |
           ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}
__device__ __forceinline__ bool mbar_wait(uint32_t bar, uint32_t parity) {
    uint32_t ok = 0;
    for (int i = 0; !ok && i < (1 << 22); ++i)
        asm volatile("{\n\t.reg .pred P;\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2;\n\tselp.u32 %0, 1, 0, P;\n\t}"
                     : "=r"(ok) : "r"(bar), "r"(parity) : "memory");
    return ok;
}

// fmt: 5 = e2m1, 4 = e3m2 (instruction-descriptor A/B format codes)
__global__ void k_check(const __grid_constant__ CUtensorMap ma, const __grid_constant__ CUtensorMap mb, uint32_t fmt,
                        uint32_t tx, float* out, int* status, int mx, int n, int sfcol) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ __align__(8) uint64_t bars[2];
    __shared__ uint32_t tmem_sh;
    const uint32_t base = ((uint32_t)__cvta_generic_to_shared(sm) + 1023) & ~1023u;
    const uint32_t sa = base, sb = base + M * 128;
    const uint32_t bfull = (uint32_t)__cvta_generic_to_shared(&bars[0]), bmma = bfull + 8;
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                         (uint32_t)__cvta_generic_to_shared(&tmem_sh)) : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bfull) : "memory");
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bmma) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = tmem_sh;
    const int warp0 = threadIdx.x >> 5;
    if (mx) {  // scale factors: 0x7F (2^0) in 8 columns of every lane
        const uint32_t v = 0x7F7F7F7Fu;
        asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1};" ::"r"(
                         tmem + ((32 * warp0) << 16) + sfcol), "r"(v) : "memory");
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t idesc = mx ? ((1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | (1u << 23) | ((uint32_t)(M >> 4) << 24))
                              : (1u << 4) | (fmt << 7) | (fmt << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
    if (threadIdx.x == 0) {
        for (int ks = 0; ks < (mx ? K / 256 : K / 128); ++ks) {
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bfull), "r"(tx)
                         : "memory");
            asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                         ::"r"(sa), "l"(&ma), "r"(ks * 128), "r"(0), "r"(bfull) : "memory");
            asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                         ::"r"(sb), "l"(&mb), "r"(ks * 128), "r"(0), "r"(bfull) : "memory");
            asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                         ::"r"(sb + 128 * 128), "l"(&mb), "r"(ks * 128), "r"(128), "r"(bfull) : "memory");
            if (!mbar_wait(bfull, ks & 1)) { *status = 1; break; }
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            for (int kk = 0; kk < 4; ++kk)
                if (mx)
                    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                                 "tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], %1, %2, %3, [%5], [%5], p;\n\t}"
                                 ::"r"(tmem), "l"(sdesc(sa + 32 * kk)), "l"(sdesc(sb + 32 * kk)), "r"(idesc),
                                 "r"((ks > 0 || kk > 0) ? 1u : 0u), "r"(tmem + sfcol));
                else
                asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::f8f6f4 [%0], %1, %2, %3, p;\n\t}"
                             ::"r"(tmem), "l"(sdesc(sa + 32 * kk)), "l"(sdesc(sb + 32 * kk)), "r"(idesc),
                             "r"((ks > 0 || kk > 0) ? 1u : 0u));
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bmma) : "memory");
            if (!mbar_wait(bmma, ks & 1)) { *status = 2; break; }  // smem reused by the next slice
        }
    }
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int c = 0; c < n; ++c) {
        uint32_t v;
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(v) : "r"(tmem + ((32 * warp) << 16) + c));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        out[(32 * warp + lane) * N + c] = __uint_as_float(v);
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
}

static uint8_t enc_e2m1(int v) {  // exact integers |v| <= 4 (and 6)
    static const int mag[7] = {0x0, 0x2, 0x4, 0x5, 0x6, -1, 0x7};
    const int a = v < 0 ? -v : v;
    return (uint8_t)(mag[a] | (v < 0 ? 0x8 : 0));
}
static uint8_t enc_e3m2(int v) {  // exact integers |v| <= 8
    static const int mag[9] = {0x00, 0x0C, 0x10, 0x12, 0x14, 0x15, 0x16, 0x17, 0x18};
    const int a = v < 0 ? -v : v;
    return (uint8_t)(mag[a] | (v < 0 ? 0x20 : 0));
}
// pack 16-element groups little-endian: element j at bit bits*j of its group
static void pack(const std::vector<int>& v, int rows, int bits, std::vector<uint8_t>& out) {
    const int gbytes = 16 * bits / 8;
    out.assign((size_t)rows * K / 16 * gbytes, 0);
    for (int r = 0; r < rows; ++r)
        for (int g = 0; g < K / 16; ++g) {
            unsigned __int128 acc = 0;
            for (int j = 0; j < 16; ++j) {
                const int x = v[(size_t)r * K + 16 * g + j];
                const unsigned __int128 code = bits == 4 ? enc_e2m1(x) : enc_e3m2(x);
                acc |= code << (bits * j);
            }
            memcpy(&out[((size_t)r * K / 16 + g) * gbytes], &acc, gbytes);
        }
}

typedef CUresult (*enc_t)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                          const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                          CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int run(int bits, int maxv, int seed, bool worst, int mx = 0, int n = N, int sfcol = 256) {
    srand(seed);
    std::vector<int> A((size_t)M * K), B((size_t)N * K);
    for (auto& x : A) x = worst ? ((rand() & 1) ? maxv : -maxv) : rand() % (2 * maxv + 1) - maxv;
    for (auto& x : B) x = worst ? ((rand() & 1) ? maxv : -maxv) : rand() % (2 * maxv + 1) - maxv;
    if (worst)  // the largest accumulated magnitude: row 0 of A equal to row 0 of B
        for (int k = 0; k < K; ++k) A[k] = B[k];
    std::vector<uint8_t> pa, pb;
    pack(A, M, bits, pa);
    pack(B, N, bits, pb);
    void *da, *db;
    float* dout;
    cudaMalloc(&da, pa.size());
    cudaMalloc(&db, pb.size());
    cudaMalloc(&dout, sizeof(float) * M * N);
    cudaMemcpy(da, pa.data(), pa.size(), cudaMemcpyHostToDevice);
    cudaMemcpy(db, pb.data(), pb.size(), cudaMemcpyHostToDevice);
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
    enc_t enc = (enc_t)p;
    CUtensorMap ma, mb;
    const CUtensorMapDataType dt = mx ? CU_TENSOR_MAP_DATA_TYPE_UINT8
                                   : bits == 4 ? CU_TENSOR_MAP_DATA_TYPE_16U4_ALIGN16B : CU_TENSOR_MAP_DATA_TYPE_16U6_ALIGN16B;
    const cuuint64_t rowbytes = (cuuint64_t)K * bits / 8;
    const cuuint64_t kdim = mx ? rowbytes : K;
    cuuint64_t da_dims[2] = {kdim, M}, db_dims[2] = {kdim, N}, strides[1] = {rowbytes};
    cuuint32_t boxa[2] = {128, M}, boxb[2] = {128, 128}, es[2] = {1, 1};
    CUresult r1 = enc(&ma, dt, 2, da, da_dims, strides, boxa, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                      CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    CUresult r2 = enc(&mb, dt, 2, db, db_dims, strides, boxb, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                      CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r1 || r2) {
        printf("encode failed %d %d\n", (int)r1, (int)r2);
        return 1;
    }
    const int smem = (M + N) * 128 + 1024;
    cudaFuncSetAttribute(k_check, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    int* dst;
    cudaMalloc(&dst, 4);
    cudaError_t e = cudaSuccess;
    int st = 0;
    // transaction bytes: shared-memory bytes written (128 per row) or global bytes read (packed)
    for (uint32_t tx : {(uint32_t)((M + N) * 128), (uint32_t)((M + N) * 128 * bits / 8)}) {
        cudaMemset(dst, 0, 4);
        cudaMemset(dout, 0, sizeof(float) * M * N);
        k_check<<<1, 128, smem>>>(ma, mb, bits == 4 ? 5u : 4u, tx, dout, dst, mx, n, sfcol);
        e = cudaDeviceSynchronize();
        cudaMemcpy(&st, dst, 4, cudaMemcpyDeviceToHost);
        printf("  tx %u bytes: %s, status %d\n", tx, cudaGetErrorString(e), st);
        if (e == cudaSuccess && st == 0) break;
    }
    std::vector<float> out((size_t)M * N);
    cudaMemcpy(out.data(), dout, sizeof(float) * M * N, cudaMemcpyDeviceToHost);
    long long bad = 0, maxabs = 0;
    double worst_err = 0;
    for (int i = 0; i < M; ++i)
        for (int j = 0; j < n; ++j) {
            long long s = 0;
            for (int k = 0; k < K; ++k) s += (long long)A[(size_t)i * K + k] * B[(size_t)j * K + k];
            maxabs = llabs(s) > maxabs ? llabs(s) : maxabs;
            const double err = (double)out[(size_t)i * N + j] - (double)s;
            if (err != 0) ++bad;
            worst_err = fabs(err) > worst_err ? fabs(err) : worst_err;
        }
    printf("%s%s bits=%d |v|<=%d %s n=%d: %s, mismatches %lld / %d, max |exact| %lld, max |err| %g, out[0]=%g\n",
           bits == 4 ? "e2m1" : "e3m2", mx ? " mxf4 packed" : "", bits, maxv, worst ? "worst-case" : "random", n,
           cudaGetErrorString(e), bad, M * n,
           maxabs, worst_err, out[0]);
    cudaFree(da);
    cudaFree(db);
    cudaFree(dout);
    return bad != 0;
}

int main() {
    int fails = 0;
    fails += run(4, 4, 1, false);
    fails += run(4, 4, 2, true);
    fails += run(6, 8, 3, false);
    fails += run(6, 8, 4, true);
    fails += run(4, 4, 5, false, 1, 256, 256);
    fails += run(4, 4, 6, true, 1, 256, 256);
    fails += run(4, 4, 7, false, 1, 240, 240);
    fails += run(4, 4, 8, true, 1, 240, 240);
    printf(fails ? "NARROW MMA NOT EXACT\n" : "NARROW MMA EXACT\n");
    return fails;
}
