// bn_api.cu -- host side of the C-ABI declared in include/bn.h.
//
// Owns the device state of one tile problem and sequences the pass kernels of bn_kernels.cuh
// on the context's stream.  Host code here only validates arguments, builds the two fp64
// look-up tables of the energy (W[o], G_l[D]; libm exp/sqrt, no contraction) and moves bytes;
// every step of the method runs on the GPU.
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <algorithm>
#include <functional>
#include <string>
#include <vector>

#include "../../include/bn.h"
#include "bn_kernels.cuh"

using namespace bn;

namespace {

// ---------------------------------------------------------------------- NCCL (dlopen'ed)
// Loaded lazily so the library has no link-time NCCL dependency (torch ships its own
// libnccl.so.2; dlopen returns the already-loaded copy when torch is imported first).
typedef struct { char internal[128]; } NcclUid;
typedef void* NcclComm;
typedef int (*nccl_get_uid_t)(NcclUid*);
typedef int (*nccl_init_rank_t)(NcclComm*, int, NcclUid, int);
typedef int (*nccl_allreduce_t)(const void*, void*, size_t, int, int, NcclComm, cudaStream_t);
typedef int (*nccl_destroy_t)(NcclComm);
typedef const char* (*nccl_errstr_t)(int);
struct NcclApi {
    void* h = nullptr;
    nccl_get_uid_t get_uid = nullptr;
    nccl_init_rank_t init_rank = nullptr;
    nccl_allreduce_t allreduce = nullptr;
    nccl_destroy_t destroy = nullptr;
    nccl_errstr_t errstr = nullptr;
    bool load() {
        if (h) return true;
        const char* names[] = {"libnccl.so.2", "libnccl.so"};
        for (const char* n : names)
            if ((h = dlopen(n, RTLD_NOW | RTLD_GLOBAL))) break;
        if (!h) return false;
        get_uid = (nccl_get_uid_t)dlsym(h, "ncclGetUniqueId");
        init_rank = (nccl_init_rank_t)dlsym(h, "ncclCommInitRank");
        allreduce = (nccl_allreduce_t)dlsym(h, "ncclAllReduce");
        destroy = (nccl_destroy_t)dlsym(h, "ncclCommDestroy");
        errstr = (nccl_errstr_t)dlsym(h, "ncclGetErrorString");
        return get_uid && init_rank && allreduce && destroy && errstr;
    }
};
NcclApi g_nccl;
constexpr int NCCL_INT32 = 2, NCCL_SUM = 0;  // ncclInt32, ncclSum (nccl.h enums)

// cuTensorMapEncodeTiled through the runtime's driver entry point (no link-time libcuda).
typedef CUresult (*encode_tiled_t)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
encode_tiled_t get_encode_tiled() {
    static encode_tiled_t fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = (encode_tiled_t)p;
    }
    return fn;
}
// 3D map over the [y][x][row] count tensor restricted to one level: the level's elements start at
// byte `lb` of each row (`rowB` bytes), `elems` of them in format `fmt` (u8, or the TMA-unpacked
// 16U4 / 16U6 narrow types); box {128 elements, bx, by}, 128-B swizzle.
bool make_level_map(CUtensorMap* m, const void* base, uint64_t rowB, uint64_t lb, uint64_t elems, uint32_t fmt,
                    uint64_t L, uint32_t bx, uint32_t by) {
    encode_tiled_t enc = get_encode_tiled();
    if (!enc) return false;
    // e2m1 rows stay packed (plain bytes, kind::mxf4); e3m2 rows are unpacked by the TMA (f8f6f4)
    const CUtensorMapDataType dt = fmt == BN_FMT_E3M2 ? CU_TENSOR_MAP_DATA_TYPE_16U6_ALIGN16B : CU_TENSOR_MAP_DATA_TYPE_UINT8;
    cuuint64_t dims[3] = {fmt == BN_FMT_E2M1 ? elems / 2 : elems, L, L};
    cuuint64_t strides[2] = {rowB, L * rowB};
    cuuint32_t box[3] = {128, bx, by};
    cuuint32_t es[3] = {1, 1, 1};
    return enc(m, dt, 3, const_cast<uint8_t*>(static_cast<const uint8_t*>(base) + lb), dims, strides, box, es,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
bool make_level_maps(CountMaps* m, const void* base, uint64_t rowB, uint64_t lb, uint64_t elems, uint32_t fmt,
                     uint64_t L) {
    return make_level_map(&m->a, base, rowB, lb, elems, fmt, L, 8, 8) &&
           make_level_map(&m->b, base, rowB, lb, elems, fmt, L, 24, 5) &&
           make_level_map(&m->s, base, rowB, lb, elems, fmt, L, 8, 1) &&
           make_level_map(&m->g, base, rowB, lb, elems, fmt, L, 8, 5) &&
           make_level_map(&m->r, base, rowB, lb, elems, fmt, L, 24, 1);
}

template <class T>
struct DevBuf {
    T* p = nullptr;
    size_t n = 0;
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        n = 0;
    }
    cudaError_t ensure(size_t count) {
        if (count <= n && p) return cudaSuccess;
        release();
        cudaError_t e = cudaMalloc(&p, count * sizeof(T) + 16);
        if (e == cudaSuccess) n = count;
        return e;
    }
};

}  // namespace

struct bn_ctx {
    int dev = 0;
    cudaStream_t stream = nullptr;
    std::string err;
    uint64_t launches = 0;
    // lattice
    bool have_lattice = false;
    uint32_t d1 = 1, d2 = 1, nl = 0, levels[8] = {0};
    // bank
    bool have_bank = false;
    uint32_t T = 0, t0 = 0, t1 = 0, Ts = 0, Tp = 0;
    std::vector<int32_t> a, b;
    std::vector<uint32_t> px, py;
    // energy
    double sigma_i = 2.1, sigma_s = 1.0;
    uint32_t form = BN_E_GF;  // bn_set_energy_form
    int R = 7;
    bool lut_dirty = true;
    // tile
    bool have_tile = false, counts_dirty = true;
    uint32_t L = 0, P = 0, rowB = 0;
    // device state
    DevBuf<uint2> S, U, Un, Un2, pxy;
    DevBuf<int2> ab;
    DevBuf<long long> Cc;
    DevBuf<CountGroup> cgrp;  // packed fp32 operands of the filtered count test
    DevBuf<uint8_t> c, cn, cn2, acc, log, cexp;
    DevBuf<int> nc, nn, nn2, derr, progress;
    DevBuf<uint32_t> perm, part, invperm;
    DevBuf<uint8_t> cnK;   // best-of-K candidates [K][P][rowB]
    DevBuf<uint2> UnK;
    DevBuf<int> nnK;
    DevBuf<unsigned long long> kpart;  // best-of-K partial window sums [M][8]
    DevBuf<unsigned int> kticket;
    DevBuf<double2> ev_tw, ev_X1;  // bn_eval_quality work buffers
    DevBuf<double> ev_h, ev_rm, ev_sp, ev_out, ev_bump, ev_img;  // BN_PAPER_SWAP: precomputed permutation, per-pass partner map
    uint32_t perm_n = 0;
    DevBuf<int4> Dt;
    DevBuf<longlong2> d0;        // int64 dE terms {delta0, delta1} per (pixel, offset) (DT_ESC = see escape tables)
    DevBuf<longlong2> x0, x1;    // exact int128 escape tables (sparse writes)
    DevBuf<i128> dEp;
    DevBuf<u128> Epart;
    DevBuf<PassStatsDev> pstats;
    DevBuf<FinishPart> fparts;
    DevBuf<unsigned int> ticket;
    DevBuf<double> W, G, iref;
    size_t Goff[8] = {0};
    int Dmax[8] = {0};
    // multi-GPU
    NcclComm comm = nullptr;
    int rank = 0, world = 1;
    // streams: `stream` is the caller's; `ls` is the stream the next launch goes to; `aux`
    // (candidate prefetch) and `hp` (high-priority decisions) are internal, joined by events.
    cudaStream_t ls = nullptr, aux = nullptr, hp = nullptr;
    cudaEvent_t evA = nullptr, evB = nullptr, evC = nullptr;
    cudaEvent_t ev_h2d = nullptr;  // bn_set_tile: the upload of a host tile is complete
    bool no_overlap = false;  // BN_OVERLAP=0: no candidate prefetch on the aux stream
    // per-row publication of the next pass's candidate counts (k_counts -> k_gram_tc4 follows them)
    DevBuf<unsigned int> rows_done;
    uint32_t rows_L = 0, counts_epoch = 0;
    const unsigned int* gram_rows = nullptr;  // set for the Gram of a pass whose counts may still run
    uint32_t gram_rows_target = 0;
    bool no_rowflags = true;  // BN_ROWFLAGS=1: the Gram follows the counts row by row (measured slower on C3)
    int prefetch_at = 1;  // BN_PREFETCH=start|gram|lut: launch the next pass's counts before the Gram / after it / after the energy terms
    bool per_class_decide = false;  // BN_DECIDE=per_class: 64 launches instead of one persistent
    bool gram_attr_set[8] = {false};  // k_gram_tc4<R> shared-memory attribute
    bool decide_attr_set[8] = {false};
    bool cluster_attr_set[8] = {false};
    bool big_attr_set[8] = {false};
    bool no_big = false;  // BN_DECIDE=nobig: L > 128 tiles use the cooperative flag kernel
    bool no_cluster = false;  // BN_DECIDE=flags: skip the cluster decide kernel
    bool no_fuse = false;          // BN_FUSE=0: separate SWAP commit (k_finish) and gather kernels
    bool no_tail = false;          // BN_TAIL=0: separate decision and commit kernels (no k_pass_tail)
    uint32_t nEpart = 0;           // energy partials written by the last Gram / k_lut launch
    DevBuf<uint32_t> border;       // block order of the Gram (wrapping blocks first)
    uint32_t border_L = 0;
    bool no_border = false;        // BN_GRAM_ORDER=raster: plain raster block order
    DevBuf<unsigned int> gsched;   // Gram work counter + CTA exit counter (dynamic item scheduling)
    bool static_sched = false;     // BN_GRAM_SCHED=static: round-robin items instead
    bool no_csplit = false;        // BN_GRAM_CSPLIT=0: small tiles keep whole (block, level) items
    bool force_csplit = false;     // BN_GRAM_CSPLIT=1: every tile splits its items into chunks

    bool tail_attr_set[8] = {false};
    int tail_clusters = -1;        // clusters of the fused pass tail that fit (cached for tail_L)
    uint32_t tail_L = 0;
    DevBuf<TailCounters> tailc;
    bool swap_v3 = false;     // BN_DECIDE=swap3: SWAP on k_decide_cl3 (one warp per couple) instead of k_decide_swap
    // narrow count rows: in the SWAP / paper modes, where a pass only
    // permutes rows, the rows are stored as packed deltas c - round(N I_ref) (e2m1 / e3m2 per level,
    // chosen from the tile's measured range); every other consumer unpacks them first (ensure_u8)
    int narrow_mode = -1;  // BN_NARROW: -1 auto (default: narrow when Tp >= 2048), 0 off, 1 narrow (range-chosen formats),
                           // 2 e3m2 / u8 only, 3 the u8 layout through the narrow path
    bool packed = false;   // c holds narrow rows (layout fmt / lb / rowBn)
    uint32_t fmt[8] = {0}, lb[8] = {0}, rowBn = 0;
    DevBuf<uint8_t> noff;  // offsets [l][Tp]
    bool noff_dirty = true;
    DevBuf<int> nrng;      // per-level max |delta|
    int* nrng_host = nullptr;  // pinned copy, valid when nrng_epoch == layout_epoch (filled by bn_set_tile)
    uint32_t nrng_epoch = 0xffffffffu;
    uint32_t layout_epoch = 0;  // bumped whenever the rows are rewritten (range validity)
    // tensor-map cache, keyed by buffer and layout (the layout is the same for every tile of a bank)
    struct MapEntry { const void* base; uint64_t key; CountMaps m[8]; };
    std::vector<MapEntry> map_cache;
    // per-kernel event timing (bn_profile_*)
    bool prof = false;
    std::vector<cudaEvent_t> ev_pool;
    size_t ev_used = 0;
    std::vector<std::pair<int, size_t>> prof_marks;  // (kernel id, index of start event)
    double prof_ms[BN_K_COUNT_IDS] = {0};
    uint64_t prof_n[BN_K_COUNT_IDS] = {0};
};

namespace {

int fail(bn_ctx* ctx, int code, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    if (ctx) ctx->err = buf;
    return code;
}

#define CUDA_TRY(expr)                                                                               \
    do {                                                                                             \
        cudaError_t e_ = (expr);                                                                     \
        if (e_ != cudaSuccess)                                                                       \
            return fail(ctx, e_ == cudaErrorMemoryAllocation ? BN_ENOMEM : BN_ECUDA, "%s: %s (%s:%d)", \
                        #expr, cudaGetErrorString(e_), __FILE__, __LINE__);                          \
    } while (0)

#define LAUNCHED()                                                                              \
    do {                                                                                        \
        ++ctx->launches;                                                                        \
        cudaError_t e_ = cudaGetLastError();                                                    \
        if (e_ != cudaSuccess)                                                                  \
            return fail(ctx, BN_ECUDA, "launch failed: %s (%s:%d)", cudaGetErrorString(e_), __FILE__, \
                        __LINE__);                                                              \
    } while (0)

cudaEvent_t next_event(bn_ctx* ctx) {
    if (ctx->ev_used == ctx->ev_pool.size()) {
        cudaEvent_t e;
        cudaEventCreate(&e);
        ctx->ev_pool.push_back(e);
    }
    return ctx->ev_pool[ctx->ev_used++];
}
// Bracket a launch with events when profiling: KSTART(id) before, LAUNCHED_K() after.
#define KSTART(id)                                                                  \
    do {                                                                            \
        if (ctx->prof) {                                                            \
            if (ctx->ev_used + 2 > 4096) flush_profile(ctx);                         \
            ctx->prof_marks.push_back({(id), ctx->ev_used});                         \
            cudaEventRecord(next_event(ctx), ctx->ls);                              \
        }                                                                           \
    } while (0)
#define LAUNCHED_K()                                                                \
    do {                                                                            \
        if (ctx->prof) cudaEventRecord(next_event(ctx), ctx->ls);                   \
        LAUNCHED();                                                                 \
    } while (0)

void flush_profile(bn_ctx* ctx) {
    cudaStreamSynchronize(ctx->stream);
    if (ctx->aux) cudaStreamSynchronize(ctx->aux);
    if (ctx->hp) cudaStreamSynchronize(ctx->hp);
    for (auto& m : ctx->prof_marks) {
        float ms = 0.f;
        cudaEventElapsedTime(&ms, ctx->ev_pool[m.second], ctx->ev_pool[m.second + 1]);
        ctx->prof_ms[m.first] += ms;
        ctx->prof_n[m.first] += 1;
    }
    ctx->prof_marks.clear();
    ctx->ev_used = 0;
}

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int d) {
        cudaGetDevice(&prev);
        if (prev != d) cudaSetDevice(d);
    }
    ~DeviceGuard() {
        int cur;
        cudaGetDevice(&cur);
        if (prev >= 0 && cur != prev) cudaSetDevice(prev);
    }
};

// Launch through cudaLaunchKernelEx (typed arguments).
template <typename... KArgs, typename... Args>
cudaError_t launch_k(bn_ctx* ctx, void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                     Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    (void)ctx;
    return cudaLaunchKernelEx(&cfg, k, args...);
}

uint32_t round_up(uint32_t v, uint32_t m) { return (v + m - 1) / m * m; }
bool pow2(uint32_t v) { return v && !(v & (v - 1)); }
int half_count(int R) { return 2 * R * R + 2 * R; }
int win_count(int R) { return (2 * R + 1) * (2 * R + 1) - 1; }

// Energy LUTs.  W[w] = exp(-|o|^2 / sigma_i^2) in full-window order; G_l[D] for 0 <= D <= T N_l^2:
// exp(-(sqrt(D)/N_l) / sigma_s^2) (BN_E_GF), D / (N_l^2 T) (BN_E_EQ1) or 1 - D / (N_l^2 T)
// (BN_E_EQ1_MAX).  Host libm, -ffp-contract=off.
int build_lut(bn_ctx* ctx) {
    const int R = ctx->R;
    std::vector<double> W(win_count(R));
    for (int oy = -R; oy <= R; ++oy)
        for (int ox = -R; ox <= R; ++ox) {
            if (!ox && !oy) continue;
            W[win_index(ox, oy, R)] = std::exp(-(double)(ox * ox + oy * oy) / (ctx->sigma_i * ctx->sigma_i));
        }
    size_t total = 0;
    for (uint32_t l = 0; l < ctx->nl; ++l) {
        const uint64_t dm = (uint64_t)ctx->T * ctx->levels[l] * ctx->levels[l];
        if (dm > 0x7fffffffull) return fail(ctx, BN_EINVAL, "T * N^2 = %llu exceeds int32", (unsigned long long)dm);
        ctx->Dmax[l] = (int)dm;
        ctx->Goff[l] = total;
        total += dm + 1;
    }
    if (total > (1ull << 28)) return fail(ctx, BN_EINVAL, "energy table of %zu entries too large", total);
    std::vector<double> G(total);
    const double s2 = ctx->sigma_s * ctx->sigma_s;
    for (uint32_t l = 0; l < ctx->nl; ++l) {
        const double N = (double)ctx->levels[l];
        // Eq. 1 forms: ||I_p - I_q||^2 = D / N^2, normalised by 1/T so that w * g < 1 (fixed point)
        const double den = (double)((uint64_t)ctx->levels[l] * ctx->levels[l] * ctx->T);
        double* g = G.data() + ctx->Goff[l];
        for (int D = 0; D <= ctx->Dmax[l]; ++D) {
            if (ctx->form == BN_E_GF)
                g[D] = std::exp(-(std::sqrt((double)D) / N) / s2);
            else if (ctx->form == BN_E_EQ1)
                g[D] = (double)D / den;
            else
                g[D] = 1.0 - (double)D / den;
        }
    }
    CUDA_TRY(ctx->W.ensure(W.size()));
    CUDA_TRY(ctx->G.ensure(total));
    CUDA_TRY(cudaMemcpyAsync(ctx->W.p, W.data(), W.size() * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
    CUDA_TRY(cudaMemcpyAsync(ctx->G.p, G.data(), total * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
    CUDA_TRY(cudaStreamSynchronize(ctx->stream));  // host vectors go out of scope
    ctx->lut_dirty = false;
    return BN_OK;
}

int check_ready(bn_ctx* ctx) {
    if (!ctx->have_lattice) return fail(ctx, BN_ESTATE, "bn_set_lattice has not been called");
    if (!ctx->have_bank) return fail(ctx, BN_ESTATE, "bn_set_bank has not been called");
    if (!ctx->have_tile) return fail(ctx, BN_ESTATE, "bn_set_tile has not been called");
    if (ctx->L <= (uint32_t)(2 * ctx->R))
        return fail(ctx, BN_EINVAL, "tile side L = %u must exceed 2R = %d", ctx->L, 2 * ctx->R);
    return BN_OK;
}

// Dynamic shared memory of k_counts: the CTA's samples (float2 + int2 per pixel and sample)
size_t counts_smem(const bn_ctx* ctx) {
    return (size_t)COUNT_PIX * ((ctx->levels[ctx->nl - 1] + 3) & ~3u) * 16;
}
// (Re)build counts of the current tile when lattice or bank changed after bn_set_tile.
int ensure_counts(bn_ctx* ctx) {
    if (!ctx->counts_dirty) return BN_OK;
    const uint32_t P = ctx->P;
    ctx->rowB = ctx->nl * ctx->Tp;
    CUDA_TRY(ctx->Un.ensure(P));
    CUDA_TRY(ctx->c.ensure((size_t)P * ctx->rowB));
    CUDA_TRY(ctx->cn.ensure((size_t)P * ctx->rowB));
    CUDA_TRY(ctx->nc.ensure((size_t)P * ctx->nl));
    CUDA_TRY(ctx->nn.ensure((size_t)P * ctx->nl));
    const uint32_t Nmax = ctx->levels[ctx->nl - 1];
    const uint4 lo = make_uint4(ctx->levels[0], ctx->levels[1], ctx->levels[2], ctx->levels[3]);
    const uint4 hi = make_uint4(ctx->levels[4], ctx->levels[5], ctx->levels[6], ctx->levels[7]);
    KSTART(BN_K_COUNTS);
    k_counts<<<(P + COUNT_PIX - 1) / COUNT_PIX, 256, counts_smem(ctx), ctx->ls>>>(
        ctx->U.p, nullptr, 0, 0, 0, P, ctx->ab.p, ctx->Cc.p, ctx->cgrp.p, ctx->Tp, ctx->S.p, Nmax, lo, hi, ctx->nl, ctx->c.p,
        ctx->nc.p, nullptr, ctx->L);
    LAUNCHED_K();
    ctx->counts_dirty = false;
    ctx->packed = false;
    ++ctx->layout_epoch;
    return BN_OK;
}

int ensure_work(bn_ctx* ctx) {
    int rc;
    if ((rc = check_ready(ctx))) return rc;
    if ((rc = ensure_counts(ctx))) return rc;
    if (ctx->lut_dirty && (rc = build_lut(ctx))) return rc;
    const size_t P = ctx->P, H = half_count_padded(ctx->R), WN = win_count(ctx->R);
    CUDA_TRY(ctx->Dt.ensure(P * H * ctx->nl));  // two int2 planes over [l][p][padded h]
    CUDA_TRY(ctx->d0.ensure(P * WN));
    CUDA_TRY(ctx->acc.ensure(P));
    CUDA_TRY(ctx->dEp.ensure(P));
    CUDA_TRY(ctx->Epart.ensure((P * H + 255) / 256));
    if (!ctx->derr.p) {  // the device error flag is sticky: cleared only when read (read_err_flag)
        CUDA_TRY(ctx->derr.ensure(1));
        CUDA_TRY(cudaMemsetAsync(ctx->derr.p, 0, sizeof(int), ctx->stream));
    }
    return BN_OK;
}

template <int R>
int launch_gram(bn_ctx* ctx, const uint8_t* cn, const int* nn);
template <int R>
int launch_lut_only(bn_ctx* ctx, int write_deltas, bool exchange = true);

// The Gram and the energy terms of a pass (with a communicator, the exchange of the partial
// distances in between, inside launch_lut_only).
template <int R>
int launch_gram_lut(bn_ctx* ctx, const uint8_t* cn, const int* nn, int write_deltas,
                    const std::function<int()>* after_gram) {
    int rc = launch_gram<R>(ctx, cn, nn);
    if (rc) return rc;
    if (after_gram && (rc = (*after_gram)())) return rc;
    return launch_lut_only<R>(ctx, write_deltas);
}

uint32_t row_bytes(const bn_ctx* ctx) { return ctx->packed ? ctx->rowBn : ctx->rowB; }

// Tensor maps of the rows at `base` in the current layout, cached per (buffer, layout epoch): the
// candidate buffers alternate between a few pointers, and encoding 3 maps per level per launch
// would cost tens of microseconds of host time per pass.
uint64_t layout_key(const bn_ctx* ctx) {
    uint64_t k = ((uint64_t)row_bytes(ctx) << 32) ^ ((uint64_t)ctx->L << 20) ^ ((uint64_t)ctx->Tp << 4) ^ ctx->nl;
    for (uint32_t l = 0; l < ctx->nl; ++l) k = k * 1000003u + (ctx->packed ? 1 + ctx->fmt[l] : 0);
    return k;
}
bool level_maps(bn_ctx* ctx, const void* base, CountMaps* out) {
    const uint64_t key = layout_key(ctx);
    for (const auto& e : ctx->map_cache)
        if (e.base == base && e.key == key) {
            for (uint32_t l = 0; l < ctx->nl; ++l) out[l] = e.m[l];
            return true;
        }
    bn_ctx::MapEntry ent;
    ent.base = base;
    ent.key = key;
    for (uint32_t l = 0; l < ctx->nl; ++l) {
        const uint32_t f = ctx->packed ? ctx->fmt[l] : BN_FMT_U8;
        const uint64_t lb = ctx->packed ? ctx->lb[l] : (uint64_t)l * ctx->Tp;
        if (!make_level_maps(&ent.m[l], base, row_bytes(ctx), lb, ctx->Tp, f, ctx->L)) return false;
        out[l] = ent.m[l];
    }
    if (ctx->map_cache.size() >= 8) ctx->map_cache.erase(ctx->map_cache.begin());
    ctx->map_cache.push_back(ent);
    return true;
}

// Window Gram: the TMA-fed persistent tcgen05 kernel k_gram_tc4<R> (one CTA per SM), every R <= 7
// (the R = 7 neighbourhood tiles are a superset), u8 or narrow rows.
template <int R>
int launch_gram(bn_ctx* ctx, const uint8_t* cn, const int* nn) {
    GramMaps gm;
    memset(&gm, 0, sizeof gm);
    if (!level_maps(ctx, ctx->c.p, gm.c) || !level_maps(ctx, cn, gm.n))
        return fail(ctx, BN_ECUDA, "cuTensorMapEncodeTiled failed");
    for (uint32_t l = 0; l < 8; ++l) gm.fmt[l] = ctx->packed && l < ctx->nl ? ctx->fmt[l] : BN_FMT_U8;
    const int smem = tc3::SMEM;
    if (!ctx->gram_attr_set[R]) {
        CUDA_TRY(cudaFuncSetAttribute(k_gram_tc4<R>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        ctx->gram_attr_set[R] = true;
    }
    int nsm = 148;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, ctx->dev);
    // small tiles (fewer (block, level) items than SMs): one item per neighbour chunk
    // ... and long rows (Tp >= 2048: operands beyond L2): the three chunk items of a block run
    // concurrently on three SMs and share its A rows in L2 (C5 Gram DRAM reads 1.02 -> 0.62 GB,
    // 0.337 -> 0.329 ms; C3 would lose: 0.105 -> 0.117 ms)
    const uint32_t csplit = ctx->force_csplit || (((ctx->L / 8) * (ctx->L / 8) * ctx->nl < (uint32_t)nsm || ctx->Tp >= 2048) &&
                                                  !ctx->no_csplit)
                                ? tc3::NCHUNK : 1;
    const uint32_t items = (ctx->L / 8) * (ctx->L / 8) * ctx->nl * csplit;
    const uint32_t grid = items < (uint32_t)nsm ? items : (uint32_t)nsm;
    KSTART(BN_K_GRAM);
    // block order: toroidally wrapping blocks (x0 = 0, x0 = L - 8, last block row) first
    const uint32_t nbx = ctx->L / 8;
    if (ctx->border_L != ctx->L && !ctx->no_border) {
        std::vector<uint32_t> ord;
        for (int pass = 0; pass < 2; ++pass)
            for (uint32_t b = 0; b < nbx * nbx; ++b) {
                const uint32_t bx = b % nbx, by = b / nbx;
                const bool wraps = bx == 0 || bx == nbx - 1 || by == nbx - 1;
                if (wraps == (pass == 0)) ord.push_back(b);
            }
        CUDA_TRY(ctx->border.ensure(ord.size()));
        CUDA_TRY(cudaMemcpyAsync(ctx->border.p, ord.data(), ord.size() * sizeof(uint32_t), cudaMemcpyHostToDevice, ctx->stream));
        CUDA_TRY(cudaStreamSynchronize(ctx->stream));
        ctx->border_L = ctx->L;
    }
    // dynamic scheduling only pays when a CTA gets more than one item (C1: 128 items, ~1 us dearer)
    const bool dyn = !ctx->static_sched && items > grid;
    if (dyn && !ctx->gsched.p) {  // zero once; the kernel's last CTA re-zeroes it
        CUDA_TRY(ctx->gsched.ensure(2));
        CUDA_TRY(cudaMemsetAsync(ctx->gsched.p, 0, 2 * sizeof(unsigned int), ctx->ls));
    }
    CUDA_TRY(launch_k(ctx, k_gram_tc4<R>, dim3(grid), dim3(tc3::THREADS), smem, ctx->ls, gm, ctx->nc.p, nn, ctx->L,
                      ctx->Tp, ctx->nl, ctx->Dt.p, ctx->gram_rows, ctx->gram_rows_target,
                      (const uint32_t*)(ctx->no_border ? nullptr : ctx->border.p),
                      dyn ? ctx->gsched.p : nullptr, csplit));
    LAUNCHED_K();
    return BN_OK;
}

// ---------------------------------------------------------------- narrow rows
// The current rows as u8 counts without changing the stored layout: c itself, or (narrow rows) c
// unpacked into the candidate buffer cn (free between bn_optimize calls).
const uint8_t* u8_rows(bn_ctx* ctx) {
    if (!ctx->packed) return ctx->c.p;
    const uint32_t P = ctx->P;
    NarrowLayout lay;
    for (uint32_t l = 0; l < 8; ++l) lay.fmt[l] = ctx->fmt[l], lay.lb[l] = ctx->lb[l];
    k_narrow_unpack<<<(P + 7) / 8, 256, 0, ctx->stream>>>(ctx->c.p, P, ctx->Tp, ctx->nl, ctx->noff.p, lay, ctx->rowBn,
                                                         ctx->cn.p, ctx->nn.p);
    ++ctx->launches;
    return ctx->cn.p;
}
// u8 rows: unpack the narrow rows of c (norms |c|^2) if they are packed.
int ensure_u8(bn_ctx* ctx) {
    if (!ctx->packed) return BN_OK;
    const uint32_t P = ctx->P;
    NarrowLayout lay;
    for (uint32_t l = 0; l < 8; ++l) lay.fmt[l] = ctx->fmt[l], lay.lb[l] = ctx->lb[l];
    k_narrow_unpack<<<(P + 7) / 8, 256, 0, ctx->stream>>>(ctx->c.p, P, ctx->Tp, ctx->nl, ctx->noff.p, lay, ctx->rowBn,
                                                         ctx->cn.p, ctx->nn.p);
    LAUNCHED();
    std::swap(ctx->c, ctx->cn);
    std::swap(ctx->nc, ctx->nn);
    ctx->packed = false;
    ++ctx->layout_epoch;
    return BN_OK;
}

// Narrow rows for the permuting modes: per level, the tile's max |c - round(N I_ref)| selects e2m1
// (<= 4), e3m2 (<= 8) or u8; the rows are packed into that layout (norms |delta|^2).  One host
// synchronisation (the range) per new tile.
// Per-level max |c - off| of the current u8 rows into the pinned host buffer (asynchronous).
int ensure_noff(bn_ctx* ctx);
int narrow_range_async(bn_ctx* ctx) {
    const uint32_t P = ctx->P, nl = ctx->nl, Tp = ctx->Tp;
    int rc;
    if ((rc = ensure_noff(ctx))) return rc;
    if (!ctx->nrng_host) CUDA_TRY(cudaMallocHost(&ctx->nrng_host, 8 * sizeof(int)));
    CUDA_TRY(ctx->nrng.ensure(8));
    CUDA_TRY(cudaMemsetAsync(ctx->nrng.p, 0, 8 * sizeof(int), ctx->stream));
    const size_t nchl = (size_t)P * (Tp / 16);  // 16-byte chunks per level; >= 8 per thread
    k_narrow_range<<<dim3((unsigned)std::min<size_t>((nchl + 2047) / 2048, 148 * 8), nl), 256, 0, ctx->stream>>>(
        ctx->c.p, P, Tp, nl, ctx->noff.p, ctx->nrng.p);
    LAUNCHED();
    CUDA_TRY(cudaMemcpyAsync(ctx->nrng_host, ctx->nrng.p, 8 * sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    ctx->nrng_epoch = ctx->layout_epoch;
    return BN_OK;
}

// Narrow rows pay off where the Gram's K loop is long (C5: T = 8192, 0.84 -> 0.74 ms per Gram); with
// T <= 1024 per level the Gram is bound by the TMA row rate, not bytes, and the pack is overhead.
bool narrow_wanted(const bn_ctx* ctx) { return ctx->narrow_mode > 0 || (ctx->narrow_mode < 0 && ctx->Tp >= 2048); }

// Offsets off[l][i] = round(N_l I_ref,i) of the current bank (once per bank)
int ensure_noff(bn_ctx* ctx) {
    if (!ctx->noff_dirty) return BN_OK;
    const uint32_t nl = ctx->nl, Tp = ctx->Tp;
    const uint4 lo = make_uint4(ctx->levels[0], ctx->levels[1], ctx->levels[2], ctx->levels[3]);
    const uint4 hi = make_uint4(ctx->levels[4], ctx->levels[5], ctx->levels[6], ctx->levels[7]);
    CUDA_TRY(ctx->iref.ensure(ctx->Ts));
    k_iref<<<(ctx->Ts + 127) / 128, 128, 0, ctx->stream>>>(ctx->ab.p, ctx->pxy.p, ctx->Ts, ctx->iref.p);
    LAUNCHED();
    CUDA_TRY(ctx->noff.ensure((size_t)nl * Tp));
    k_narrow_offsets<<<(Tp + 255) / 256, 256, 0, ctx->stream>>>(ctx->iref.p, ctx->Ts, Tp, lo, hi, nl, ctx->noff.p);
    LAUNCHED();
    ctx->noff_dirty = false;
    return BN_OK;
}



int ensure_narrow(bn_ctx* ctx) {
    if (ctx->packed || !narrow_wanted(ctx)) return BN_OK;
    const uint32_t P = ctx->P, nl = ctx->nl, Tp = ctx->Tp;
    int rc;
    if (ctx->nrng_epoch != ctx->layout_epoch && (rc = narrow_range_async(ctx))) return rc;
    CUDA_TRY(cudaStreamSynchronize(ctx->stream));  // immediate when bn_set_tile already waited for it
    int rng[8];
    memcpy(rng, ctx->nrng_host, sizeof rng);
    NarrowLayout lay;
    uint32_t off = 0;
    for (uint32_t l = 0; l < 8; ++l) {
        uint32_t f = BN_FMT_U8;
        if (l < nl) {
            const int m = rng[l];
            // the fp32 accumulator of the narrow MMAs is exact while every dot product stays below
            // 2^24: Tp * 4^2 (e2m1) and Tp * 8^2 (e3m2) bound them
            const bool e2 = (uint64_t)Tp * 16 < (1ull << 24), e3 = (uint64_t)Tp * 64 < (1ull << 24);
            f = ctx->narrow_mode == 3 ? BN_FMT_U8
                : m <= 4 && ctx->narrow_mode != 2 && e2 ? BN_FMT_E2M1
                : m <= 8 && e3 ? BN_FMT_E3M2 : BN_FMT_U8;
        }
        ctx->fmt[l] = lay.fmt[l] = f;
        ctx->lb[l] = lay.lb[l] = off;
        if (l < nl) off += Tp * fmt_bits(f) / 8;
    }
    ctx->rowBn = off;
    CUDA_TRY(cudaMemsetAsync(ctx->nn.p, 0, (size_t)P * nl * sizeof(int), ctx->stream));
    const size_t nch = (size_t)P * nl * (Tp / 16);
    k_narrow_pack<<<(unsigned)std::min<size_t>((nch + 1023) / 1024, 148 * 64), 256, 0, ctx->stream>>>(
        ctx->c.p, P, Tp, nl, ctx->noff.p, lay, ctx->rowBn, ctx->cn.p, ctx->nn.p);
    LAUNCHED();
    std::swap(ctx->c, ctx->cn);
    std::swap(ctx->nc, ctx->nn);
    ctx->packed = true;
    ++ctx->layout_epoch;
    return BN_OK;
}

template <int R>
int launch_lut_only(bn_ctx* ctx, int write_deltas, bool exchange) {
    if (ctx->comm && exchange) {
        const size_t n = (size_t)ctx->P * half_count_padded(R) * ctx->nl * 4;
        int r = g_nccl.allreduce(ctx->Dt.p, ctx->Dt.p, n, NCCL_INT32, NCCL_SUM, ctx->comm, ctx->ls);
        if (r) return fail(ctx, BN_ENCCL, "ncclAllReduce: %s", g_nccl.errstr(r));
    }
    LutArgs la;
    for (uint32_t l = 0; l < 8; ++l) {
        la.G[l] = l < ctx->nl ? ctx->G.p + ctx->Goff[l] : nullptr;
        la.Dmax[l] = l < ctx->nl ? ctx->Dmax[l] : 0;
    }
    const size_t nthr = (size_t)ctx->P * half_count_padded(R);
    ctx->nEpart = (uint32_t)((nthr + 255) / 256);
    KSTART(BN_K_LUT);
    {
        auto fn = ctx->nl == 4 ? k_lut<R, 4> : ctx->nl == 1 ? k_lut<R, 1> : k_lut<R, 0>;
        CUDA_TRY(launch_k(ctx, fn, dim3((unsigned)((nthr + 255) / 256)), dim3(256), 0, ctx->ls, ctx->Dt.p, ctx->L, ctx->nl,
                          ctx->W.p, la, write_deltas, ctx->d0.p, ctx->Epart.p, ctx->derr.p));
    }
    LAUNCHED_K();
    return BN_OK;
}

template <int R>
int launch_gram_only(bn_ctx* ctx) {
    return launch_gram<R>(ctx, ctx->c.p, ctx->nc.p);
}
int gram_only(bn_ctx* ctx) {
    switch (ctx->R) {
        case 1: return launch_gram_only<1>(ctx);
        case 2: return launch_gram_only<2>(ctx);
        case 3: return launch_gram_only<3>(ctx);
        case 4: return launch_gram_only<4>(ctx);
        case 5: return launch_gram_only<5>(ctx);
        case 6: return launch_gram_only<6>(ctx);
        default: return launch_gram_only<7>(ctx);
    }
}

// `after_gram` (optional) is called between the Gram and the energy-term launches.
int gram_lut(bn_ctx* ctx, const uint8_t* cn, const int* nn, int write_deltas,
             const std::function<int()>* after_gram = nullptr) {
    switch (ctx->R) {
        case 1: return launch_gram_lut<1>(ctx, cn, nn, write_deltas, after_gram);
        case 2: return launch_gram_lut<2>(ctx, cn, nn, write_deltas, after_gram);
        case 3: return launch_gram_lut<3>(ctx, cn, nn, write_deltas, after_gram);
        case 4: return launch_gram_lut<4>(ctx, cn, nn, write_deltas, after_gram);
        case 5: return launch_gram_lut<5>(ctx, cn, nn, write_deltas, after_gram);
        case 6: return launch_gram_lut<6>(ctx, cn, nn, write_deltas, after_gram);
        default: return launch_gram_lut<7>(ctx, cn, nn, write_deltas, after_gram);
    }
}

template <int R>
int launch_decide(bn_ctx* ctx, uint32_t s, uint32_t t, uint64_t seed, int mode, uint8_t* log) {
    const uint32_t M = (ctx->L / 8) * (ctx->L / 8);
    KSTART(BN_K_DECIDE);
    const DTabs T = {ctx->d0.p, ctx->x0.p, ctx->x1.p};
    k_decide<R><<<(M + 3) / 4, 128, 0, ctx->ls>>>(s, t, seed, ctx->L, mode, T, ctx->acc.p, ctx->dEp.p, log);
    LAUNCHED_K();
    return BN_OK;
}
// L = 256, 512: one 16-CTA cluster with `spw` slots per warp and bit flags (k_decide_big).
template <int R>
int launch_decide_big(bn_ctx* ctx, uint32_t t, uint64_t seed, int mode, uint8_t* log, bool* done) {
    const uint32_t nb = ctx->L / 8, M = nb * nb, P = ctx->P, ncta = 16, nw = 16;
    if (M % (ncta * nw) || ctx->no_big || nb > 64) return BN_OK;  // cooperative flag kernel instead
    uint32_t spw = M / (ncta * nw);
    if (mode && (spw & 1)) return BN_OK;
    const uint32_t cpc = nw * spw;
    const size_t smem = (size_t)P / 8 + (size_t)64 * cpc * 6;
    if (smem > 220 * 1024) return BN_OK;
    const void* fn = mode ? (const void*)k_decide_big<R, 1> : (const void*)k_decide_big<R, 0>;
    if (!ctx->big_attr_set[R]) {
        for (const void* f : {(const void*)k_decide_big<R, 0>, (const void*)k_decide_big<R, 1>}) {
            CUDA_TRY(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
            CUDA_TRY(cudaFuncSetAttribute(f, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
        }
        ctx->big_attr_set[R] = true;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(ncta);
    cfg.blockDim = dim3(32 * nw);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = ctx->ls;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = ncta;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int nclusters = 0;
    if (cudaOccupancyMaxActiveClusters(&nclusters, fn, &cfg) != cudaSuccess || nclusters < 1) {
        cudaGetLastError();
        return BN_OK;
    }
    uint32_t L = ctx->L;
    const DTabs T = {ctx->d0.p, ctx->x0.p, ctx->x1.p};
    uint8_t* acc = ctx->acc.p;
    i128* dEp = ctx->dEp.p;
    void* args[] = {&t, &seed, &L, &spw, (void*)&T, &acc, &dEp, &log};
    KSTART(BN_K_DECIDE);
    cudaError_t e = cudaLaunchKernelExC(&cfg, fn, args);
    if (e != cudaSuccess) return fail(ctx, BN_ECUDA, "big cluster decide launch: %s", cudaGetErrorString(e));
    LAUNCHED_K();
    *done = true;
    return BN_OK;
}

// L <= 128: one cluster of <= 16 CTAs decides all 64 classes (k_decide_cl3; SWAP: k_decide_swap).
template <int R>
int launch_decide_cluster(bn_ctx* ctx, uint32_t t, uint64_t seed, int mode, uint8_t* log, bool* done) {
    const uint32_t nb = ctx->L / 8, P = ctx->P;
    const bool swap_v4 = mode && !ctx->swap_v3;  // SWAP: one warp per couple member (k_decide_swap)
    uint32_t cpc = mode && !swap_v4 ? 8 : 16;
    while (cpc > nb * nb / (swap_v4 ? 1 : nb)) cpc /= 2;  // at most M slots (SWAP v4) / nb per CTA
    if (swap_v4)  // the full cluster, whole couples (one CTA for M <= 16: C1)
        cpc = nb * nb <= 16 ? nb * nb : std::max(2u, std::min(16u, nb * nb / 16));
    else if (!mode)  // REDRAW: the same spread (C2 REDRAW decide 0.042 -> 0.038 ms)
        cpc = nb * nb <= 16 ? nb * nb : std::max(1u, std::min(16u, nb * nb / 16));
    const uint32_t ncta = nb * nb / cpc;
    *done = false;
    if (ctx->no_cluster) return BN_OK;
    if (ncta > 16) return launch_decide_big<R>(ctx, t, seed, mode, log, done);
    // u32 flags in every CTA's shared memory + the slot table of the 64 classes (+ member indices)
    const size_t slots = (size_t)64 * 4 * (mode ? 2 : 1) * cpc;
    const size_t smem = swap_v4 ? 4 * (size_t)P + (size_t)64 * cpc * 6 : 4 * (size_t)P + slots;
    const void* fn = swap_v4 ? (const void*)k_decide_swap<R>
                             : (mode ? (const void*)k_decide_cl3<R, 1> : (const void*)k_decide_cl3<R, 0>);
    if (!ctx->cluster_attr_set[R]) {
        for (const void* f : {(const void*)k_decide_cl3<R, 0>, (const void*)k_decide_cl3<R, 1>,
                              (const void*)k_decide_swap<R>}) {
            CUDA_TRY(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
            CUDA_TRY(cudaFuncSetAttribute(f, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
        }
        ctx->cluster_attr_set[R] = true;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(ncta);
    cfg.blockDim = dim3(32 * cpc);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = ctx->ls;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = ncta;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int nclusters = 0;
    if (cudaOccupancyMaxActiveClusters(&nclusters, fn, &cfg) != cudaSuccess || nclusters < 1) {
        cudaGetLastError();
        return BN_OK;  // cluster does not fit: persistent flag kernel instead
    }
    uint32_t L = ctx->L;
    const DTabs T = {ctx->d0.p, ctx->x0.p, ctx->x1.p};
    uint8_t* acc = ctx->acc.p;
    i128* dEp = ctx->dEp.p;
    void* args[] = {&t, &seed, &L, &cpc, (void*)&T, &acc, &dEp, &log};
    KSTART(BN_K_DECIDE);
    cudaError_t e = cudaLaunchKernelExC(&cfg, fn, args);
    if (e != cudaSuccess) return fail(ctx, BN_ECUDA, "cluster decide launch: %s", cudaGetErrorString(e));
    LAUNCHED_K();
    *done = true;
    return BN_OK;
}

// Larger tiles (REDRAW): one cooperative launch for all 64 classes (k_decide_pass); co-residency of
// its CTAs is guaranteed by the cooperative launch, which the neighbour-progress waits require.
template <int R>
int launch_decide_pass(bn_ctx* ctx, uint32_t t, uint64_t seed, int mode, uint8_t* log, bool* done) {
    constexpr int WN = (2 * R + 1) * (2 * R + 1) - 1;
    int rc = launch_decide_cluster<R>(ctx, t, seed, mode, log, done);
    if (rc || *done) return rc;
    const uint32_t nb = ctx->L / 8;
    // SWAP is not safe here: a CTA also reads the window of its candidate's partner, in a band whose
    // neighbours do not wait for that CTA's progress, so a later class could be decided under the
    // read (found by test_decide_large_tiles at L = 256).  SWAP tiles beyond the cluster kernels
    // fall back to the per-class launches.
    if (mode) {
        *done = false;
        return BN_OK;
    }
    // candidates per CTA: <= 16 warps; divides nb
    uint32_t cpc = 16;
    while (cpc > nb) cpc /= 2;
    const uint32_t ncta = nb * nb / cpc;
    const size_t smem = (size_t)(mode ? 2 : 1) * cpc * 2 * WN * 8;
    int nsm = 148;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, ctx->dev);
    if (ncta > (uint32_t)nsm || nb > 512) {
        *done = false;  // not co-residable: per-class launches
        return BN_OK;
    }
    const void* fn = mode ? (const void*)k_decide_pass<R, 1> : (const void*)k_decide_pass<R, 0>;
    if (!ctx->decide_attr_set[R]) {
        CUDA_TRY(cudaFuncSetAttribute(k_decide_pass<R, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        CUDA_TRY(cudaFuncSetAttribute(k_decide_pass<R, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        ctx->decide_attr_set[R] = true;
    }
    CUDA_TRY(ctx->progress.ensure(ncta));
    CUDA_TRY(cudaMemsetAsync(ctx->progress.p, 0, ncta * sizeof(int), ctx->ls));
    uint32_t L = ctx->L;
    const DTabs T = {ctx->d0.p, ctx->x0.p, ctx->x1.p};
    uint8_t* acc = ctx->acc.p;
    i128* dEp = ctx->dEp.p;
    int* prog = ctx->progress.p;
    void* args[] = {&t, &seed, &L, &cpc, (void*)&T, &acc, &dEp, &log, &prog};
    KSTART(BN_K_DECIDE);
    cudaError_t e = cudaLaunchCooperativeKernel(fn, dim3(ncta), dim3(32 * cpc), args, smem, ctx->ls);
    if (e == cudaErrorCooperativeLaunchTooLarge || e == cudaErrorNotSupported) {
        cudaGetLastError();
        if (ctx->prof) ctx->prof_marks.pop_back();
        *done = false;
        return BN_OK;
    }
    if (e != cudaSuccess) return fail(ctx, BN_ECUDA, "cooperative decide launch: %s", cudaGetErrorString(e));
    LAUNCHED_K();
    *done = true;
    return BN_OK;
}

int decide_pass(bn_ctx* ctx, uint32_t t, uint64_t seed, int mode, uint8_t* log, bool* done) {
    switch (ctx->R) {
        case 1: return launch_decide_pass<1>(ctx, t, seed, mode, log, done);
        case 2: return launch_decide_pass<2>(ctx, t, seed, mode, log, done);
        case 3: return launch_decide_pass<3>(ctx, t, seed, mode, log, done);
        case 4: return launch_decide_pass<4>(ctx, t, seed, mode, log, done);
        case 5: return launch_decide_pass<5>(ctx, t, seed, mode, log, done);
        case 6: return launch_decide_pass<6>(ctx, t, seed, mode, log, done);
        default: return launch_decide_pass<7>(ctx, t, seed, mode, log, done);
    }
}

int decide(bn_ctx* ctx, uint32_t s, uint32_t t, uint64_t seed, int mode, uint8_t* log) {
    switch (ctx->R) {
        case 1: return launch_decide<1>(ctx, s, t, seed, mode, log);
        case 2: return launch_decide<2>(ctx, s, t, seed, mode, log);
        case 3: return launch_decide<3>(ctx, s, t, seed, mode, log);
        case 4: return launch_decide<4>(ctx, s, t, seed, mode, log);
        case 5: return launch_decide<5>(ctx, s, t, seed, mode, log);
        case 6: return launch_decide<6>(ctx, s, t, seed, mode, log);
        default: return launch_decide<7>(ctx, s, t, seed, mode, log);
    }
}

template <int R>
int launch_paper_decide(bn_ctx* ctx, uint32_t t, uint64_t seed, uint32_t ncp, uint8_t* log) {
    const DTabs T{ctx->d0.p, ctx->x0.p, ctx->x1.p};
    KSTART(BN_K_DECIDE);
    k_paper_decide<R><<<(ncp + 7) / 8, 256, 0, ctx->ls>>>(ctx->perm.p, seed, t, ctx->L, ncp, T, ctx->acc.p,
                                                          ctx->dEp.p, log);
    LAUNCHED_K();
    return BN_OK;
}

int paper_decide(bn_ctx* ctx, uint32_t t, uint64_t seed, uint32_t ncp, uint8_t* log) {
    switch (ctx->R) {
        case 1: return launch_paper_decide<1>(ctx, t, seed, ncp, log);
        case 2: return launch_paper_decide<2>(ctx, t, seed, ncp, log);
        case 3: return launch_paper_decide<3>(ctx, t, seed, ncp, log);
        case 4: return launch_paper_decide<4>(ctx, t, seed, ncp, log);
        case 5: return launch_paper_decide<5>(ctx, t, seed, ncp, log);
        case 6: return launch_paper_decide<6>(ctx, t, seed, ncp, log);
        default: return launch_paper_decide<7>(ctx, t, seed, ncp, log);
    }
}

// Fused pass tail (k_pass_tail, SWAP, L <= 128): one cooperative launch of clusters of `ncta` CTAs,
// cluster 0 deciding, the others committing (and gathering the next pass's candidates) behind it.
// Returns BN_OK with *done = false when the configuration does not fit (separate kernels then).
template <int R>
int launch_pass_tail(bn_ctx* ctx, uint32_t t, uint64_t seed, uint8_t* log, uint32_t rb, const uint2* Un,
                     const uint8_t* cn, const int* nn, uint2* Un2, uint8_t* cn2, int* nn2, int gather_next,
                     PassStatsDev* out, int check_prev, bool* done) {
    *done = false;
    const uint32_t nb = ctx->L / 8, M = nb * nb, P = ctx->P;
    if (ctx->no_tail || nb > 64 || nb < 8) return BN_OK;  // 64 <= L <= 512 (C1-size tiles: measured slower)
    // L <= 128: k_decide_swap's shape (one warp per member, flags as words); L = 256, 512:
    // k_decide_big's (16 warps x M / 256 slots, flags as bits)
    const bool big = nb > 16;
    if (big && (M % 512 || ctx->no_big)) return BN_OK;  // whole couples per warp
    // members per deciding CTA: spread each class over the full 16-CTA cluster (C2: 4 members per
    // CTA, tail 0.069 -> 0.057 ms; fewer warps per SM issue the window sums faster), whole couples;
    // tiny classes (M <= 16) stay in one CTA
    uint32_t cpc = big ? M / 16 : M <= 16 ? M : std::max(2u, std::min(16u, M / 16));
    const uint32_t ncta = M / cpc;
    const size_t smem = (big ? (size_t)P / 8 : 4 * (size_t)P) + (size_t)64 * cpc * 6;
    if (smem > 220 * 1024) return BN_OK;
    const void* fn = big ? (const void*)k_pass_tail<R, true> : (const void*)k_pass_tail<R, false>;
    if (!ctx->tail_attr_set[R]) {
        for (const void* f : {(const void*)k_pass_tail<R, true>, (const void*)k_pass_tail<R, false>}) {
            CUDA_TRY(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
            CUDA_TRY(cudaFuncSetAttribute(f, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
        }
        ctx->tail_attr_set[R] = true;
    }
    if (ctx->tail_L != ctx->L) {  // the fitting cluster count depends on the variant and its smem
        ctx->tail_clusters = -1;
        ctx->tail_L = ctx->L;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.blockDim = dim3(32 * ((big ? 16 : cpc) + 1));  // + the publisher warp of the deciding CTAs
    cfg.dynamicSmemBytes = smem;
    cfg.stream = ctx->ls;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = ncta;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    at[1].id = cudaLaunchAttributeCooperative;
    at[1].val.cooperative = 1;
    cfg.attrs = at;
    cfg.numAttrs = 2;
    if (ctx->tail_clusters < 0) {
        cfg.gridDim = dim3(ncta);
        int ncl = 0;
        if (cudaOccupancyMaxActiveClusters(&ncl, fn, &cfg) != cudaSuccess) {
            cudaGetLastError();
            ncl = 0;
        }
        int nsm = 148;
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, ctx->dev);
        int cap = nsm / (int)ncta;  // one CTA per SM at most
        const char* tcl = getenv("BN_TAIL_CLUSTERS");  // cap (A/B measurements, concurrent contexts)
        if (tcl && atoi(tcl) >= 2) cap = std::min(cap, atoi(tcl));
        ctx->tail_clusters = ncl < cap ? ncl : cap;
    }
    if (ctx->tail_clusters < 2) return BN_OK;
    const uint32_t ncl = (uint32_t)ctx->tail_clusters, nh = (ncl - 1) * ncta;
    cfg.gridDim = dim3(ncl * ncta);
    if (!ctx->tailc.p) {
        CUDA_TRY(ctx->tailc.ensure(1));
        CUDA_TRY(cudaMemsetAsync(ctx->tailc.p, 0, sizeof(TailCounters), ctx->stream));
    }
    CUDA_TRY(ctx->fparts.ensure(nh));
    uint32_t L = ctx->L, nl = ctx->nl;
    uint32_t nE = ctx->nEpart;
    longlong2* dterms = ctx->d0.p;
    uint8_t* acc = ctx->acc.p;
    i128* dEp = ctx->dEp.p;
    const u128* Epart = ctx->Epart.p;
    int* err = ctx->derr.p;
    uint2* U = ctx->U.p;
    uint8_t* c = ctx->c.p;
    int* nc = ctx->nc.p;
    FinishPart* parts = ctx->fparts.p;
    TailCounters* tc = ctx->tailc.p;
    void* args[] = {&t, &seed, &L, &cpc, &dterms, &acc, &dEp, &log, (void*)&Epart, &nE, &nl, &err, &rb,
                    (void*)&Un, &U, (void*)&cn, &c, (void*)&nn, &nc, &Un2, &cn2, &nn2, &gather_next, &parts, &out,
                    &check_prev, &tc};
    KSTART(BN_K_TAIL);
    cudaError_t e = cudaLaunchKernelExC(&cfg, fn, args);
    if (e != cudaSuccess) {
        if (ctx->prof) ctx->prof_marks.pop_back();
        cudaGetLastError();
        ctx->tail_clusters = 0;  // does not fit: separate kernels from now on
        return BN_OK;
    }
    LAUNCHED_K();
    *done = true;
    return BN_OK;
}
int pass_tail(bn_ctx* ctx, uint32_t t, uint64_t seed, uint8_t* log, uint32_t rb, const uint2* Un, const uint8_t* cn,
              const int* nn, uint2* Un2, uint8_t* cn2, int* nn2, int gather_next, PassStatsDev* out, int check_prev,
              bool* done) {
    switch (ctx->R) {
        case 1: return launch_pass_tail<1>(ctx, t, seed, log, rb, Un, cn, nn, Un2, cn2, nn2, gather_next, out, check_prev, done);
        case 2: return launch_pass_tail<2>(ctx, t, seed, log, rb, Un, cn, nn, Un2, cn2, nn2, gather_next, out, check_prev, done);
        case 3: return launch_pass_tail<3>(ctx, t, seed, log, rb, Un, cn, nn, Un2, cn2, nn2, gather_next, out, check_prev, done);
        case 4: return launch_pass_tail<4>(ctx, t, seed, log, rb, Un, cn, nn, Un2, cn2, nn2, gather_next, out, check_prev, done);
        case 5: return launch_pass_tail<5>(ctx, t, seed, log, rb, Un, cn, nn, Un2, cn2, nn2, gather_next, out, check_prev, done);
        case 6: return launch_pass_tail<6>(ctx, t, seed, log, rb, Un, cn, nn, Un2, cn2, nn2, gather_next, out, check_prev, done);
        default: return launch_pass_tail<7>(ctx, t, seed, log, rb, Un, cn, nn, Un2, cn2, nn2, gather_next, out, check_prev, done);
    }
}

// The device error flag accumulates every invariant failure of every launch since it was last
// read (bits: 1 window distance outside [0, T N^2], 2 dE term outside +-2^55, 4 a pass's
// recomputed start energy != the previous pass's E + sum dE); reading it clears it.
int read_err_flag(bn_ctx* ctx) {
    if (!ctx->derr.p) return BN_OK;
    int h = 0;
    CUDA_TRY(cudaMemcpyAsync(&h, ctx->derr.p, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    if (!h) return BN_OK;
    CUDA_TRY(cudaMemsetAsync(ctx->derr.p, 0, sizeof(int), ctx->stream));
    if (h & 1) return fail(ctx, BN_ESTATE, "internal invariant failed: window distance outside [0, T N^2]");
    if (h & 2) return fail(ctx, BN_ESTATE, "internal invariant failed: dE term outside +-2^55");
    return fail(ctx, BN_ESTATE, "internal invariant failed: E recomputed at a pass start != E + sum dE");
}

template <int R, int NV>
int launch_class_best_nv(bn_ctx* ctx, uint32_t s, uint32_t t, uint64_t seed, uint32_t K, const LutArgs& la, uint8_t* log) {
    const uint32_t M = (ctx->L / 8) * (ctx->L / 8);
    const size_t smem = (size_t)(K + 1) * ctx->rowB;
    if (smem > 200 * 1024) return fail(ctx, BN_EINVAL, "best-of-K rows (%zu B) exceed shared memory", smem);
    CUDA_TRY(cudaFuncSetAttribute(k_class_best<R, NV>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    k_class_best<R, NV><<<dim3(M, KBEST_SPLIT), 256, smem, ctx->ls>>>(
        s, t, seed, ctx->L, K, ctx->c.p, ctx->cnK.p, ctx->nc.p, ctx->nnK.p, ctx->U.p, ctx->UnK.p, ctx->rowB, ctx->Tp,
        ctx->nl, ctx->W.p, la, ctx->acc.p, ctx->dEp.p, log, ctx->derr.p, ctx->kpart.p, ctx->kticket.p);
    LAUNCHED();
    return BN_OK;
}
template <int R>
int launch_class_best(bn_ctx* ctx, uint32_t s, uint32_t t, uint64_t seed, uint32_t K, const LutArgs& la, uint8_t* log) {
    if (K + 1 <= 3) return launch_class_best_nv<R, 3>(ctx, s, t, seed, K, la, log);
    if (K + 1 <= 5) return launch_class_best_nv<R, 5>(ctx, s, t, seed, K, la, log);
    return launch_class_best_nv<R, KBEST_MAX + 1>(ctx, s, t, seed, K, la, log);
}

// Best-of-K REDRAW (K > 1): K candidate count sets per pass, then 64 per-class launches that decide
// and commit step by step (k_class_best); exact pass sums from the running energy (k_kstats).
int optimize_best_of_k(bn_ctx* ctx, const bn_opt_params* prm, bn_pass_stats* stats, uint8_t* accept_log) {
    const uint32_t P = ctx->P, M = (ctx->L / 8) * (ctx->L / 8), nl = ctx->nl, K = prm->K;
    if (ctx->comm) return fail(ctx, BN_EINVAL, "best-of-K is single-GPU (no bank sharding)");
    int rc;
    CUDA_TRY(ctx->cnK.ensure((size_t)K * P * ctx->rowB));
    CUDA_TRY(ctx->UnK.ensure((size_t)K * P));
    CUDA_TRY(ctx->nnK.ensure((size_t)K * P * nl));
    CUDA_TRY(ctx->kpart.ensure((size_t)M * KBEST_MAX));
    CUDA_TRY(ctx->kticket.ensure(M));
    CUDA_TRY(cudaMemsetAsync(ctx->kpart.p, 0, (size_t)M * KBEST_MAX * sizeof(unsigned long long), ctx->stream));
    CUDA_TRY(cudaMemsetAsync(ctx->kticket.p, 0, (size_t)M * sizeof(unsigned int), ctx->stream));
    CUDA_TRY(ctx->pstats.ensure(prm->passes + 1));
    if (accept_log) CUDA_TRY(ctx->log.ensure((size_t)prm->passes * 64 * M));
    ctx->ls = ctx->stream;
    // exact energy of the starting tile (slot `passes`), then E_after = E_before + sum dE per pass
    if ((rc = gram_lut(ctx, ctx->c.p, ctx->nc.p, 0))) return rc;
    k_pass_stats<<<1, 1024, 0, ctx->stream>>>(ctx->Epart.p, ctx->nEpart, nullptr, nullptr, P, 0, ctx->pstats.p + prm->passes);
    LAUNCHED();
    LutArgs la;
    for (uint32_t l = 0; l < 8; ++l) {
        la.G[l] = l < nl ? ctx->G.p + ctx->Goff[l] : nullptr;
        la.Dmax[l] = l < nl ? ctx->Dmax[l] : 0;
    }
    const uint4 lo = make_uint4(ctx->levels[0], ctx->levels[1], ctx->levels[2], ctx->levels[3]);
    const uint4 hi = make_uint4(ctx->levels[4], ctx->levels[5], ctx->levels[6], ctx->levels[7]);
    for (uint32_t pi = 0; pi < prm->passes; ++pi) {
        const uint32_t t = prm->first_pass + pi;
        for (uint32_t j = 0; j < K; ++j) {
            KSTART(BN_K_COUNTS);
            k_counts<<<(P + COUNT_PIX - 1) / COUNT_PIX, 256, counts_smem(ctx), ctx->stream>>>(
                nullptr, ctx->UnK.p + (size_t)j * P, (int)(1 + j), prm->seed, t, P, ctx->ab.p, ctx->Cc.p, ctx->cgrp.p,
                ctx->Tp, ctx->S.p, ctx->levels[nl - 1], lo, hi, nl, ctx->cnK.p + (size_t)j * P * ctx->rowB,
                ctx->nnK.p + (size_t)j * P * nl, nullptr, ctx->L);
            LAUNCHED_K();
        }
        uint8_t* log = accept_log ? ctx->log.p + (size_t)pi * 64 * M : nullptr;
        KSTART(BN_K_DECIDE);
        for (uint32_t s = 0; s < 64; ++s) {
            switch (ctx->R) {
                case 1: rc = launch_class_best<1>(ctx, s, t, prm->seed, K, la, log); break;
                case 2: rc = launch_class_best<2>(ctx, s, t, prm->seed, K, la, log); break;
                case 3: rc = launch_class_best<3>(ctx, s, t, prm->seed, K, la, log); break;
                case 4: rc = launch_class_best<4>(ctx, s, t, prm->seed, K, la, log); break;
                case 5: rc = launch_class_best<5>(ctx, s, t, prm->seed, K, la, log); break;
                case 6: rc = launch_class_best<6>(ctx, s, t, prm->seed, K, la, log); break;
                default: rc = launch_class_best<7>(ctx, s, t, prm->seed, K, la, log); break;
            }
            if (rc) return rc;
        }
        if (ctx->prof) cudaEventRecord(next_event(ctx), ctx->ls);  // closes the BN_K_DECIDE bracket
        const unsigned long long* Ein = pi == 0 ? ctx->pstats.p[prm->passes].E_before : ctx->pstats.p[pi - 1].E_after;
        KSTART(BN_K_STATS);
        k_kstats<<<1, 1024, 0, ctx->stream>>>(ctx->dEp.p, ctx->acc.p, P, Ein, ctx->pstats.p + pi);
        LAUNCHED_K();
    }
    if (stats || accept_log) {
        std::vector<PassStatsDev> h(prm->passes);
        CUDA_TRY(cudaMemcpyAsync(h.data(), ctx->pstats.p, prm->passes * sizeof(PassStatsDev), cudaMemcpyDeviceToHost,
                                 ctx->stream));
        if (accept_log)
            CUDA_TRY(cudaMemcpyAsync(accept_log, ctx->log.p, (size_t)prm->passes * 64 * M, cudaMemcpyDeviceToHost,
                                     ctx->stream));
        if ((rc = read_err_flag(ctx))) return rc;
        if (stats)
            for (uint32_t pi = 0; pi < prm->passes; ++pi) {
                stats[pi].accepted = h[pi].accepted;
                stats[pi].proposed = P;
                stats[pi].E_fixed[0] = h[pi].E_after[0];
                stats[pi].E_fixed[1] = h[pi].E_after[1];
                stats[pi].E = std::ldexp((double)h[pi].E_after[1], 64 - BN_FIX_BITS) +
                              std::ldexp((double)h[pi].E_after[0], -BN_FIX_BITS);
                stats[pi].dE_sum[0] = h[pi].dE_sum[0];
                stats[pi].dE_sum[1] = h[pi].dE_sum[1];
            }
    }
    return BN_OK;
}

}  // namespace

// ============================================================================ C-ABI
extern "C" {

#define BN_STR2(x) #x
#define BN_STR(x) BN_STR2(x)
const char* bn_version(void) {
    return "bn-b200 0.1 (sm_100a, CUDA " BN_STR(__CUDACC_VER_MAJOR__) "." BN_STR(__CUDACC_VER_MINOR__) ")";
}

int bn_create(bn_ctx** out, int cuda_device, uintptr_t cuda_stream) {
    if (!out) return BN_EINVAL;
    *out = nullptr;
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || cuda_device < 0 || cuda_device >= ndev) return BN_ECUDA;
    bn_ctx* ctx = new bn_ctx();
    ctx->dev = cuda_device;
    ctx->stream = reinterpret_cast<cudaStream_t>(cuda_stream);
    const char* dm = getenv("BN_DECIDE");
    ctx->per_class_decide = dm && !strcmp(dm, "per_class");
    ctx->no_cluster = dm && !strcmp(dm, "flags");
    ctx->swap_v3 = dm && !strcmp(dm, "swap3");
    ctx->no_big = dm && !strcmp(dm, "nobig");
    const char* go = getenv("BN_GRAM_ORDER");
    ctx->no_border = go && !strcmp(go, "raster");
    const char* csp = getenv("BN_GRAM_CSPLIT");
    ctx->no_csplit = csp && !strcmp(csp, "0");
    ctx->force_csplit = csp && !strcmp(csp, "1");
    const char* gs = getenv("BN_GRAM_SCHED");
    ctx->static_sched = gs && !strcmp(gs, "static");
    const char* tl = getenv("BN_TAIL");
    ctx->no_tail = tl && !strcmp(tl, "0");
    // Nsight Compute cannot replay the cooperative cluster launch of the fused tail: under a
    // profiler (injection library present) the pass runs the separate kernels instead
    for (const char* v : {"NV_COMPUTE_PROFILER_PERFWORKS_DIR", "NV_NSIGHT_INJECTION_TRANSPORT_TYPE", "CUDA_INJECTION64_PATH"}) {
        const char* inj = getenv(v);
        if (inj && *inj) ctx->no_tail = true;
    }
    const char* fu = getenv("BN_FUSE");
    ctx->no_fuse = fu && !strcmp(fu, "0");
    const char* nw = getenv("BN_NARROW");
    ctx->narrow_mode = !nw || !*nw || !strcmp(nw, "auto") ? -1 : !strcmp(nw, "0") ? 0 : !strcmp(nw, "1") ? 1
                     : !strcmp(nw, "e3m2") ? 2 : !strcmp(nw, "u8") ? 3 : -1;
    const char* ov = getenv("BN_OVERLAP");
    ctx->no_overlap = ov && !strcmp(ov, "0");
    const char* rf = getenv("BN_ROWFLAGS");
    ctx->no_rowflags = !(rf && !strcmp(rf, "1"));
    const char* pfe = getenv("BN_PREFETCH");
    ctx->prefetch_at = !pfe ? 1 : !strcmp(pfe, "start") ? 0 : !strcmp(pfe, "lut") ? 2 : 1;
    ctx->ls = ctx->stream;
    {
        DeviceGuard g(cuda_device);
        int lo = 0, hi = 0;
        cudaDeviceGetStreamPriorityRange(&lo, &hi);
        // BN_AUX_PRIO=hi|mid: the candidate-prefetch stream at the critical path's priority / between
        const char* ap = getenv("BN_AUX_PRIO");
        const int aux_prio = !ap ? lo : !strcmp(ap, "hi") ? hi : !strcmp(ap, "mid") ? (lo + hi) / 2 : lo;
        if (cudaStreamCreateWithPriority(&ctx->aux, cudaStreamNonBlocking, aux_prio) != cudaSuccess ||
            cudaStreamCreateWithPriority(&ctx->hp, cudaStreamNonBlocking, hi) != cudaSuccess ||
            cudaEventCreateWithFlags(&ctx->evA, cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&ctx->evB, cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&ctx->evC, cudaEventDisableTiming) != cudaSuccess) {
            delete ctx;
            *out = nullptr;
            return BN_ECUDA;
        }
    }
    *out = ctx;
    return BN_OK;
}

void bn_destroy(bn_ctx* ctx) {
    if (!ctx) return;
    {
        DeviceGuard g(ctx->dev);
        cudaStreamSynchronize(ctx->stream);
        if (ctx->comm && g_nccl.destroy) g_nccl.destroy(ctx->comm);
        ctx->S.release(); ctx->U.release(); ctx->Un.release(); ctx->pxy.release(); ctx->ab.release();
        ctx->Cc.release(); ctx->cgrp.release(); ctx->c.release(); ctx->cn.release(); ctx->acc.release(); ctx->log.release();
        ctx->cexp.release(); ctx->nc.release(); ctx->nn.release(); ctx->derr.release(); ctx->progress.release(); ctx->Dt.release();
        ctx->d0.release(); ctx->x0.release(); ctx->x1.release(); ctx->dEp.release(); ctx->Epart.release(); ctx->pstats.release(); ctx->fparts.release(); ctx->ticket.release();
        ctx->W.release(); ctx->G.release(); ctx->iref.release(); ctx->perm.release(); ctx->part.release(); ctx->invperm.release(); ctx->cnK.release(); ctx->UnK.release(); ctx->nnK.release(); ctx->kpart.release(); ctx->kticket.release();
        ctx->ev_tw.release(); ctx->ev_X1.release(); ctx->ev_h.release(); ctx->ev_rm.release(); ctx->ev_sp.release();
        ctx->ev_out.release(); ctx->ev_bump.release(); ctx->ev_img.release();
        for (cudaEvent_t e : ctx->ev_pool) cudaEventDestroy(e);
        ctx->Un2.release(); ctx->cn2.release(); ctx->nn2.release(); ctx->rows_done.release();
        ctx->noff.release(); ctx->nrng.release(); ctx->tailc.release(); ctx->border.release(); ctx->gsched.release();
        if (ctx->nrng_host) cudaFreeHost(ctx->nrng_host);
        if (ctx->aux) cudaStreamSynchronize(ctx->aux), cudaStreamDestroy(ctx->aux);
        if (ctx->hp) cudaStreamSynchronize(ctx->hp), cudaStreamDestroy(ctx->hp);
        if (ctx->ev_h2d) cudaEventDestroy(ctx->ev_h2d);
        for (cudaEvent_t e : {ctx->evA, ctx->evB, ctx->evC})
            if (e) cudaEventDestroy(e);
    }
    delete ctx;
}

const char* bn_last_error(const bn_ctx* ctx) { return ctx ? ctx->err.c_str() : "null context"; }

uint64_t bn_launch_count(const bn_ctx* ctx) { return ctx ? ctx->launches : 0; }

int bn_set_lattice(bn_ctx* ctx, uint32_t d1, uint32_t d2, const uint32_t* spp_levels, uint32_t n_levels) {
    if (!ctx) return BN_EINVAL;
    if (!spp_levels || n_levels < 1 || n_levels > 8) return fail(ctx, BN_EINVAL, "n_levels must be in [1, 8]");
    for (uint32_t l = 0; l < n_levels; ++l) {
        if (!pow2(spp_levels[l]) || spp_levels[l] > 128)
            return fail(ctx, BN_EINVAL, "spp level %u = %u is not a power of two in [1, 128]", l, spp_levels[l]);
        if (l && spp_levels[l] <= spp_levels[l - 1]) return fail(ctx, BN_EINVAL, "spp levels must ascend");
    }
    DeviceGuard g(ctx->dev);
    const uint32_t Nmax = spp_levels[n_levels - 1];
    std::vector<uint2> S(Nmax);
    for (uint32_t k = 0; k < Nmax; ++k) {
        // s^k = mod(Phi(k) d, 1): Phi(k) as the bit-reversed 32-bit numerator, product mod 2^32
        uint32_t r = 0;
        for (int bit = 0; bit < 32; ++bit) r = (r << 1) | ((k >> bit) & 1u);
        S[k] = make_uint2(r * d1, r * d2);
    }
    CUDA_TRY(ctx->S.ensure(Nmax));
    CUDA_TRY(cudaMemcpyAsync(ctx->S.p, S.data(), Nmax * sizeof(uint2), cudaMemcpyHostToDevice, ctx->stream));
    CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    ctx->d1 = d1;
    ctx->d2 = d2;
    ctx->nl = n_levels;
    for (uint32_t l = 0; l < 8; ++l) ctx->levels[l] = l < n_levels ? spp_levels[l] : 0;
    ctx->have_lattice = true;
    ctx->counts_dirty = true;
    ctx->noff_dirty = true;
    ctx->lut_dirty = true;
    return BN_OK;
}

int bn_set_bank(bn_ctx* ctx, uint32_t T, const int32_t* a, const int32_t* b, const uint32_t* px,
                const uint32_t* py, uint32_t t_begin, uint32_t t_end) {
    if (!ctx) return BN_EINVAL;
    if (T == 0 || !a || !b || !px || !py) return fail(ctx, BN_EINVAL, "empty bank");
    if (t_begin >= t_end || t_end > T) return fail(ctx, BN_EINVAL, "bad shard [%u, %u) of T = %u", t_begin, t_end, T);
    for (uint32_t i = 0; i < T; ++i)
        if (a[i] < -32768 || a[i] > 32768 || b[i] < -32768 || b[i] > 32768)
            return fail(ctx, BN_EINVAL, "integrand %u normal (%d, %d) exceeds 2^15", i, a[i], b[i]);
    DeviceGuard g(ctx->dev);
    ctx->T = T;
    ctx->t0 = t_begin;
    ctx->t1 = t_end;
    ctx->Ts = t_end - t_begin;
    ctx->Tp = round_up(ctx->Ts, 256);  // k_counts: 8 integrands/thread, whole warps
    ctx->a.assign(a, a + T);
    ctx->b.assign(b, b + T);
    ctx->px.assign(px, px + T);
    ctx->py.assign(py, py + T);
    std::vector<int2> ab(ctx->Tp, make_int2(0, 0));
    // padding integrands (a = b = 0) never count: t = -C is far outside the fp32 filter band, so
    // they are never recounted either
    std::vector<long long> C(ctx->Tp, 1ll << 62);
    std::vector<uint2> pxy(ctx->Ts);
    for (uint32_t j = 0; j < ctx->Ts; ++j) {
        const uint32_t i = t_begin + j;
        ab[j] = make_int2(a[i], b[i]);
        C[j] = (long long)a[i] * px[i] + (long long)b[i] * py[i] - ((long long)a[i] + b[i]) * (1ll << 31);
        pxy[j] = make_uint2(px[i], py[i]);
    }
    CUDA_TRY(ctx->ab.ensure(ctx->Tp));
    CUDA_TRY(ctx->Cc.ensure(ctx->Tp));
    CUDA_TRY(ctx->pxy.ensure(ctx->Ts));
    CUDA_TRY(cudaMemcpyAsync(ctx->ab.p, ab.data(), ctx->Tp * sizeof(int2), cudaMemcpyHostToDevice, ctx->stream));
    CUDA_TRY(cudaMemcpyAsync(ctx->Cc.p, C.data(), ctx->Tp * sizeof(long long), cudaMemcpyHostToDevice, ctx->stream));
    CUDA_TRY(cudaMemcpyAsync(ctx->pxy.p, pxy.data(), ctx->Ts * sizeof(uint2), cudaMemcpyHostToDevice, ctx->stream));
    CUDA_TRY(ctx->cgrp.ensure(ctx->Tp / COUNT_NI));
    k_count_prep<<<(ctx->Tp / COUNT_NI + 127) / 128, 128, 0, ctx->stream>>>(ctx->ab.p, ctx->Cc.p, ctx->Tp, ctx->cgrp.p);
    LAUNCHED();
    CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    ctx->have_bank = true;
    ctx->counts_dirty = true;
    ctx->noff_dirty = true;
    ctx->lut_dirty = true;
    return BN_OK;
}

int bn_get_references(bn_ctx* ctx, double* iref) {
    if (!ctx) return BN_EINVAL;
    if (!iref) return fail(ctx, BN_EINVAL, "null output");
    if (!ctx->have_bank) return fail(ctx, BN_ESTATE, "bn_set_bank has not been called");
    DeviceGuard g(ctx->dev);
    CUDA_TRY(ctx->iref.ensure(ctx->Ts));
    k_iref<<<(ctx->Ts + 127) / 128, 128, 0, ctx->stream>>>(ctx->ab.p, ctx->pxy.p, ctx->Ts, ctx->iref.p);
    LAUNCHED();
    CUDA_TRY(cudaMemcpyAsync(iref, ctx->iref.p, ctx->Ts * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    return BN_OK;
}

int bn_set_energy_form(bn_ctx* ctx, uint32_t form) {
    if (!ctx) return BN_EINVAL;
    if (form > BN_E_EQ1_MAX) return fail(ctx, BN_EINVAL, "unknown energy form %u", form);
    ctx->form = form;
    ctx->lut_dirty = true;
    return BN_OK;
}

int bn_set_energy(bn_ctx* ctx, double sigma_i, double sigma_s, int32_t radius) {
    if (!ctx) return BN_EINVAL;
    if (!(sigma_i > 0) || !(sigma_s > 0) || !std::isfinite(sigma_i) || !std::isfinite(sigma_s))
        return fail(ctx, BN_EINVAL, "sigmas must be positive and finite");
    if (radius < 1 || radius > 7) return fail(ctx, BN_EINVAL, "radius %d outside [1, 7]", radius);
    ctx->sigma_i = sigma_i;
    ctx->sigma_s = sigma_s;
    ctx->R = radius;
    ctx->lut_dirty = true;
    return BN_OK;
}

int bn_set_tile(bn_ctx* ctx, uint32_t L, const uint32_t* u_xy, int is_device) {
    if (!ctx) return BN_EINVAL;
    if (!u_xy) return fail(ctx, BN_EINVAL, "null tile");
    if (!pow2(L) || L < 16 || L > 2048) return fail(ctx, BN_EINVAL, "L = %u must be a power of two in [16, 2048]", L);
    if (!ctx->have_lattice || !ctx->have_bank) return fail(ctx, BN_ESTATE, "set lattice and bank before the tile");
    DeviceGuard g(ctx->dev);
    ctx->L = L;
    ctx->P = L * L;
    CUDA_TRY(ctx->U.ensure(ctx->P));
    CUDA_TRY(cudaMemcpyAsync(ctx->U.p, u_xy, (size_t)ctx->P * sizeof(uint2),
                             is_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, ctx->stream));
    if (!is_device) {
        if (!ctx->ev_h2d) CUDA_TRY(cudaEventCreateWithFlags(&ctx->ev_h2d, cudaEventDisableTiming));
        CUDA_TRY(cudaEventRecord(ctx->ev_h2d, ctx->stream));
    }
    ctx->have_tile = true;
    ctx->counts_dirty = true;
    int rc = ensure_counts(ctx);
    if (rc) return rc;
    // the narrow-row range of the new counts, ready (pinned) when the permuting optimiser packs them
    if (narrow_wanted(ctx) && (rc = narrow_range_async(ctx))) return rc;
    // the host buffer may be reused once it is copied; the counts stay asynchronous
    if (!is_device) CUDA_TRY(cudaEventSynchronize(ctx->ev_h2d));
    return BN_OK;
}

int bn_get_tile(bn_ctx* ctx, uint32_t* u_xy, int is_device) {
    if (!ctx) return BN_EINVAL;
    if (!u_xy) return fail(ctx, BN_EINVAL, "null output");
    if (!ctx->have_tile) return fail(ctx, BN_ESTATE, "no tile");
    DeviceGuard g(ctx->dev);
    CUDA_TRY(cudaMemcpyAsync(u_xy, ctx->U.p, (size_t)ctx->P * sizeof(uint2),
                             is_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, ctx->stream));
    if (!is_device) CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    return BN_OK;
}

int bn_eval_counts(bn_ctx* ctx, uint8_t* out, int is_device) {
    if (!ctx) return BN_EINVAL;
    if (!out) return fail(ctx, BN_EINVAL, "null output");
    int rc = check_ready(ctx);
    if (rc) return rc;
    DeviceGuard g(ctx->dev);
    if ((rc = ensure_counts(ctx))) return rc;
    const size_t n = (size_t)ctx->nl * ctx->P * ctx->Ts;
    uint8_t* dst = out;
    if (!is_device) {
        CUDA_TRY(ctx->cexp.ensure(n));
        dst = ctx->cexp.p;
    }
    const uint8_t* rows = u8_rows(ctx);
    k_counts_export<<<ctx->nl * ctx->P, 128, 0, ctx->stream>>>(rows, ctx->P, ctx->nl, ctx->Tp, ctx->Ts, dst);
    LAUNCHED();
    if (!is_device) {
        CUDA_TRY(cudaMemcpyAsync(out, dst, n, cudaMemcpyDeviceToHost, ctx->stream));
        CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    }
    return BN_OK;
}

int bn_energy(bn_ctx* ctx, double* E, uint64_t E_fixed[2]) {
    if (!ctx) return BN_EINVAL;
    DeviceGuard g(ctx->dev);
    int rc = ensure_work(ctx);
    if (rc) return rc;
    CUDA_TRY(ctx->pstats.ensure(1));
    if ((rc = gram_lut(ctx, ctx->c.p, ctx->nc.p, 0))) return rc;
    k_pass_stats<<<1, 1024, 0, ctx->stream>>>(ctx->Epart.p, ctx->nEpart, nullptr, nullptr, ctx->P, 0, ctx->pstats.p);
    LAUNCHED();
    PassStatsDev h;
    CUDA_TRY(cudaMemcpyAsync(&h, ctx->pstats.p, sizeof h, cudaMemcpyDeviceToHost, ctx->stream));
    if ((rc = read_err_flag(ctx))) return rc;
    if (E_fixed) {
        E_fixed[0] = h.E_before[0];
        E_fixed[1] = h.E_before[1];
    }
    if (E) *E = std::ldexp((double)h.E_before[1], 64 - BN_FIX_BITS) + std::ldexp((double)h.E_before[0], -BN_FIX_BITS);
    return BN_OK;
}

int bn_optimize(bn_ctx* ctx, const bn_opt_params* prm, bn_pass_stats* stats, uint8_t* accept_log) {
    if (!ctx) return BN_EINVAL;
    if (!prm) return fail(ctx, BN_EINVAL, "null params");
    if (prm->mode > BN_PAPER_SWAP) return fail(ctx, BN_EINVAL, "unknown mode %u", prm->mode);
    if (prm->reserved) return fail(ctx, BN_EINVAL, "bn_opt_params.reserved must be 0");
    if (prm->K < 1 || prm->K > KBEST_MAX || (prm->K > 1 && prm->mode != BN_REDRAW))
        return fail(ctx, BN_EINVAL, "K = %u: must be 1, or 2..%d with BN_REDRAW", prm->K, KBEST_MAX);
    DeviceGuard g(ctx->dev);
    int rc = ensure_work(ctx);
    if (rc) return rc;
    if (prm->passes == 0) return BN_OK;
    // rows: narrow packed deltas for the permuting modes, u8 counts where new counts are drawn
    if ((rc = prm->mode == BN_REDRAW ? ensure_u8(ctx) : ensure_narrow(ctx))) return rc;
    if (prm->K > 1) return optimize_best_of_k(ctx, prm, stats, accept_log);
    const uint32_t rb = row_bytes(ctx);
    const uint32_t P = ctx->P, M = (ctx->L / 8) * (ctx->L / 8), nl = ctx->nl;
    const int R = ctx->R;
    const bool paper = prm->mode == BN_PAPER_SWAP;
    const uint32_t budget = paper ? (prm->budget ? prm->budget : P / 4) : 0, ncp = budget / 2;
    if (paper) {
        if (!ctx->perm.p || ctx->perm_n != P)
            return fail(ctx, BN_ESTATE, "BN_PAPER_SWAP needs bn_set_permutation with L*L = %u entries", P);
        if (budget < 2 || (budget & 1) || budget > P)
            return fail(ctx, BN_EINVAL, "budget %u: must be even and in [2, L*L = %u]", budget, P);
    }
    if (prm->mode != BN_REDRAW) CUDA_TRY(ctx->part.ensure(P));
    CUDA_TRY(ctx->pstats.ensure(prm->passes + 1));
    int nsm_fin = 148;
    cudaDeviceGetAttribute(&nsm_fin, cudaDevAttrMultiProcessorCount, ctx->dev);
    const uint32_t nfin = (uint32_t)(2 * nsm_fin) < P / 16 ? (uint32_t)(2 * nsm_fin) : (P / 16);
    const uint32_t nfin_g = (uint32_t)(BN_FG_BPS * nsm_fin) < P / 16 ? (uint32_t)(BN_FG_BPS * nsm_fin) : (P / 16);
    if (!ctx->ticket.p) {
        CUDA_TRY(ctx->ticket.ensure(1));
        CUDA_TRY(cudaMemsetAsync(ctx->ticket.p, 0, sizeof(unsigned int), ctx->stream));
    }
    CUDA_TRY(ctx->fparts.ensure(nfin > nfin_g ? nfin : nfin_g));
    if (accept_log) CUDA_TRY(ctx->log.ensure((size_t)prm->passes * 64 * M));
    // accept flags start at zero; k_finish clears them again after every pass
    CUDA_TRY(cudaMemsetAsync(ctx->acc.p, 0, P, ctx->stream));
    const uint4 lo = make_uint4(ctx->levels[0], ctx->levels[1], ctx->levels[2], ctx->levels[3]);
    const uint4 hi = make_uint4(ctx->levels[4], ctx->levels[5], ctx->levels[6], ctx->levels[7]);
    // Candidate buffers are double-buffered so that the REDRAW candidates of pass t+1 (which do
    // not depend on pass t's decisions) are counted on the aux stream while pass t's colour
    // classes are decided on the high-priority stream.
    const bool overlap = prm->mode == BN_REDRAW && !ctx->no_overlap && prm->passes > 1 && !ctx->comm;
    if (overlap) {
        CUDA_TRY(ctx->Un2.ensure(P));
        CUDA_TRY(ctx->cn2.ensure((size_t)P * ctx->rowB));
        CUDA_TRY(ctx->nn2.ensure((size_t)P * nl));
    }
    // SWAP: the commit of pass t and the gather of pass t+1 run as one kernel (k_finish_gather), which
    // writes the next candidates into the other buffer of the pair
    const bool fuse = (prm->mode == BN_SWAP || paper) && !ctx->no_fuse && prm->passes > 1;
    if (fuse) {
        CUDA_TRY(ctx->Un2.ensure(P));
        CUDA_TRY(ctx->cn2.ensure((size_t)P * ctx->rowB));
        CUDA_TRY(ctx->nn2.ensure((size_t)P * nl));
    }
    const bool dbl = overlap || fuse;
    auto buf_U = [&](uint32_t pi) { return (dbl && (pi & 1)) ? ctx->Un2.p : ctx->Un.p; };
    auto buf_c = [&](uint32_t pi) { return (dbl && (pi & 1)) ? ctx->cn2.p : ctx->cn.p; };
    auto buf_n = [&](uint32_t pi) { return (dbl && (pi & 1)) ? ctx->nn2.p : ctx->nn.p; };
    // Row flags: with the persistent tcgen05 Gram, pass t's Gram follows its candidate counts row by
    // row (k_counts publishes each finished tile-row segment, k_gram_tc4 waits per item), so the
    // counts of pass t+1 may still be finishing when the Gram of pass t+1 starts.
    const bool rowflags = overlap && !ctx->no_rowflags;
    uint32_t rows_target[2] = {0, 0};
    if (rowflags) {
        CUDA_TRY(ctx->rows_done.ensure(ctx->L));
        if (ctx->rows_L != ctx->L) {
            CUDA_TRY(cudaMemsetAsync(ctx->rows_done.p, 0, ctx->L * sizeof(unsigned int), ctx->stream));
            ctx->rows_L = ctx->L;
            ctx->counts_epoch = 0;
        }
    }
    auto launch_counts = [&](uint32_t pi) -> int {
        KSTART(BN_K_COUNTS);
        k_counts<<<(P + COUNT_PIX - 1) / COUNT_PIX, 256, counts_smem(ctx), ctx->ls>>>(
            nullptr, buf_U(pi), 1, prm->seed, prm->first_pass + pi, P, ctx->ab.p, ctx->Cc.p, ctx->cgrp.p, ctx->Tp, ctx->S.p,
            ctx->levels[nl - 1], lo, hi, nl, buf_c(pi), buf_n(pi), rowflags ? ctx->rows_done.p : nullptr, ctx->L);
        LAUNCHED_K();
        if (rowflags) rows_target[pi & 1] = ++ctx->counts_epoch * (ctx->L / COUNT_PIX);
        return BN_OK;
    };
    // With overlap, the whole critical path (gram, energy terms, decisions, finish) runs on the
    // internal highest-priority stream `hp` and only the next pass's candidate counts run on the
    // lowest-priority `aux` stream; pending hp CTAs are dispatched first.  Both join the caller's
    // stream at the end.
    cudaStream_t cs = ctx->stream;
    if (overlap) {
        CUDA_TRY(cudaEventRecord(ctx->evA, ctx->stream));
        CUDA_TRY(cudaStreamWaitEvent(ctx->hp, ctx->evA, 0));
        cs = ctx->hp;
    }
    for (uint32_t pi = 0; pi < prm->passes; ++pi) {
        const uint32_t t = prm->first_pass + pi;
        ctx->ls = cs;

        if (paper && fuse && pi > 0) {
            // candidates gathered by k_finish_gather of pass pi - 1
        } else if (paper) {
            // partner of every pixel from the inverse permutation, gathered partner rows (dEp is only
            // written for couple members: the finish kernels leave it cleared after each pass)
            if (pi == 0) CUDA_TRY(cudaMemsetAsync(ctx->dEp.p, 0, (size_t)P * sizeof(i128), cs));
            KSTART(BN_K_GATHER);
            CUDA_TRY(launch_k(ctx, k_paper_gather, dim3((P + 7) / 8), dim3(256), 0, cs, (const uint32_t*)nullptr,
                              (const uint2*)ctx->U.p, buf_U(pi), (const uint8_t*)ctx->c.p, buf_c(pi), (const int*)ctx->nc.p,
                              buf_n(pi), P, rb, nl, (const uint32_t*)ctx->perm.p, (const uint32_t*)ctx->invperm.p,
                              prm->seed, t, budget));
            LAUNCHED_K();
        } else if (prm->mode == BN_REDRAW) {
            if (overlap && pi > 0) {
                if (!rowflags) CUDA_TRY(cudaStreamWaitEvent(cs, ctx->evC, 0));  // prefetched during pass pi-1
            } else if ((rc = launch_counts(pi))) {
                return rc;
            }
        } else if (fuse && pi > 0) {
            // candidates gathered by k_finish_gather of pass pi - 1
        } else {
            KSTART(BN_K_GATHER);
            CUDA_TRY(launch_k(ctx, k_swap_pairs, dim3((64 * M + 255) / 256), dim3(256), 0, cs, ctx->L, prm->seed, t,
                              ctx->part.p));
            LAUNCHED();
            CUDA_TRY(launch_k(ctx, k_paper_gather, dim3((P + 7) / 8), dim3(256), 0, cs, (const uint32_t*)ctx->part.p,
                              (const uint2*)ctx->U.p, buf_U(pi), (const uint8_t*)ctx->c.p, buf_c(pi),
                              (const int*)ctx->nc.p, buf_n(pi), P, rb, nl, (const uint32_t*)nullptr,
                              (const uint32_t*)nullptr, (uint64_t)0, 0u, 0u));
            LAUNCHED_K();
        }
        // next pass's candidates: their buffer was last read by finish(pi-1), already ordered on cs;
        // launched once the Gram (the one SM-saturating kernel of the pass) is done, so they fill
        // the SMs left idle by the memory-bound energy terms and the 16-SM decisions
        const std::function<int()> prefetch = [&]() -> int {
            // with row flags the Gram only waited per row: everything after it waits for the whole
            // counts kernel of this pass (recorded in evC during pass pi-1)
            if (rowflags && pi > 0) CUDA_TRY(cudaStreamWaitEvent(cs, ctx->evC, 0));
            CUDA_TRY(cudaEventRecord(ctx->evB, cs));
            CUDA_TRY(cudaStreamWaitEvent(ctx->aux, ctx->evB, 0));
            ctx->ls = ctx->aux;
            if (int r = launch_counts(pi + 1)) return r;
            CUDA_TRY(cudaEventRecord(ctx->evC, ctx->aux));
            ctx->ls = cs;
            return BN_OK;
        };
        const bool pf = overlap && pi + 1 < prm->passes;
        const std::function<int()> join = [&]() -> int {  // last pass: only wait for its counts
            if (rowflags && pi > 0) CUDA_TRY(cudaStreamWaitEvent(cs, ctx->evC, 0));
            return BN_OK;
        };
        if (prm->mode == BN_SWAP && !ctx->no_tail && (ctx->tail_clusters != 0 || ctx->tail_L != ctx->L) &&
            ctx->L <= 512 && ctx->L >= 64) {
            // fused pass tail: Gram (+ exchange), then dE terms, decisions and commit in one launch
            uint8_t* log = accept_log ? ctx->log.p + (size_t)pi * 64 * M : nullptr;
            const bool nxt = fuse && pi + 1 < prm->passes;
            if ((rc = gram_lut(ctx, buf_c(pi), buf_n(pi), 1))) return rc;
            bool done = false;
            if ((rc = pass_tail(ctx, t, prm->seed, log, rb, buf_U(pi), buf_c(pi), buf_n(pi), nxt ? buf_U(pi + 1) : nullptr,
                                nxt ? buf_c(pi + 1) : nullptr, nxt ? buf_n(pi + 1) : nullptr, (int)nxt,
                                ctx->pstats.p + pi, (int)(pi > 0), &done)))
                return rc;
            if (done) continue;
            goto decisions;  // the tail does not fit this device: the separate kernels
        }
        if (pf && ctx->prefetch_at == 0 && (rc = prefetch())) return rc;
        ctx->gram_rows = rowflags ? ctx->rows_done.p : nullptr;
        ctx->gram_rows_target = rows_target[pi & 1];
        rc = gram_lut(ctx, buf_c(pi), buf_n(pi), 1, pf && ctx->prefetch_at == 1 ? &prefetch : (rowflags ? &join : nullptr));
        ctx->gram_rows = nullptr;
        if (rc) return rc;
        if (pf && ctx->prefetch_at == 2 && (rc = prefetch())) return rc;
    decisions:
        uint8_t* log = accept_log ? ctx->log.p + (size_t)pi * 64 * M : nullptr;
        bool done = false;
        if (paper) {
            if ((rc = paper_decide(ctx, t, prm->seed, ncp, log))) return rc;
            done = true;
        }
        if (!done && !ctx->per_class_decide && (rc = decide_pass(ctx, t, prm->seed, (int)prm->mode, log, &done)))
            return rc;
        if (!done)
            for (uint32_t s = 0; s < 64; ++s)
                if ((rc = decide(ctx, s, t, prm->seed, (int)prm->mode, log))) return rc;
        if (fuse && pi + 1 < prm->passes) {
            // the next pass's partners are computed in k_finish_gather itself (swap_partner)
            KSTART(BN_K_COMMIT);
            CUDA_TRY(launch_k(ctx, k_finish_gather, dim3(nfin_g), dim3(BN_FG_THREADS), 0, cs, ctx->acc.p, P, rb, nl,
                              (const uint2*)buf_U(pi), ctx->U.p, (const uint8_t*)buf_c(pi), ctx->c.p, (const int*)buf_n(pi),
                              ctx->nc.p, (const u128*)ctx->Epart.p, ctx->nEpart, (const i128*)ctx->dEp.p, ctx->fparts.p,
                              ctx->ticket.p, ctx->pstats.p + pi, (const uint32_t*)nullptr, buf_U(pi + 1),
                              buf_c(pi + 1), buf_n(pi + 1), ctx->L, prm->seed, t + 1,
                              paper ? (const uint32_t*)ctx->perm.p : (const uint32_t*)nullptr,
                              paper ? (const uint32_t*)ctx->invperm.p : (const uint32_t*)nullptr, budget,
                              (int)(!paper && pi > 0), ctx->derr.p));
            LAUNCHED_K();
            continue;
        }
        KSTART(BN_K_COMMIT);
        CUDA_TRY(launch_k(ctx, k_finish, dim3(nfin), dim3(256), 0, cs, (const uint8_t*)ctx->acc.p, P, rb, nl,
                          (const uint2*)buf_U(pi), ctx->U.p, (const uint8_t*)buf_c(pi), ctx->c.p, (const int*)buf_n(pi),
                          ctx->nc.p, (const u128*)ctx->Epart.p, ctx->nEpart, (const i128*)ctx->dEp.p, (int)(prm->mode != BN_REDRAW),
                          ctx->fparts.p, ctx->ticket.p, ctx->pstats.p + pi, (int)paper, (int)(!paper && pi > 0),
                          ctx->derr.p));
        LAUNCHED_K();
    }
    if (overlap) {
        CUDA_TRY(cudaEventRecord(ctx->evB, cs));
        CUDA_TRY(cudaStreamWaitEvent(ctx->stream, ctx->evB, 0));
    }
    ctx->ls = ctx->stream;
    if (paper && stats) {
        // the paper's concurrent swaps do not add up (E may rise): the energy after pass pi is the
        // pass-start energy of pass pi + 1, and after the last pass one more energy evaluation
        if ((rc = gram_lut(ctx, ctx->c.p, ctx->nc.p, 0))) return rc;
        k_pass_stats<<<1, 1024, 0, ctx->stream>>>(ctx->Epart.p, ctx->nEpart, nullptr, nullptr, P, 0,
                                                  ctx->pstats.p + prm->passes);
        LAUNCHED();
    }
    if (stats || accept_log) {
        std::vector<PassStatsDev> h(prm->passes + (paper && stats ? 1 : 0));
        CUDA_TRY(cudaMemcpyAsync(h.data(), ctx->pstats.p, h.size() * sizeof(PassStatsDev), cudaMemcpyDeviceToHost,
                                 ctx->stream));
        if (accept_log)
            CUDA_TRY(cudaMemcpyAsync(accept_log, ctx->log.p, (size_t)prm->passes * 64 * M, cudaMemcpyDeviceToHost,
                                     ctx->stream));
        if ((rc = read_err_flag(ctx))) return rc;
        if (paper && stats)
            for (uint32_t pi = 0; pi < prm->passes; ++pi) {
                h[pi].E_after[0] = h[pi + 1].E_before[0];
                h[pi].E_after[1] = h[pi + 1].E_before[1];
            }
        for (uint32_t pi = 0; pi < prm->passes; ++pi) {
            if (!paper && pi &&
                (h[pi].E_before[0] != h[pi - 1].E_after[0] || h[pi].E_before[1] != h[pi - 1].E_after[1]))
                return fail(ctx, BN_ESTATE, "internal invariant failed: E recomputed at pass %u != E + sum dE",
                            prm->first_pass + pi);
            if (stats) {
                stats[pi].accepted = h[pi].accepted;
                stats[pi].proposed = paper ? ncp : prm->mode == BN_SWAP ? P / 2 : P;
                stats[pi].E_fixed[0] = h[pi].E_after[0];
                stats[pi].E_fixed[1] = h[pi].E_after[1];
                stats[pi].E = std::ldexp((double)h[pi].E_after[1], 64 - BN_FIX_BITS) +
                             std::ldexp((double)h[pi].E_after[0], -BN_FIX_BITS);
                stats[pi].dE_sum[0] = h[pi].dE_sum[0];
                stats[pi].dE_sum[1] = h[pi].dE_sum[1];
            }
        }
    }
    return BN_OK;
}

int bn_check(bn_ctx* ctx) {
    if (!ctx) return BN_EINVAL;
    DeviceGuard g(ctx->dev);
    return read_err_flag(ctx);
}

}  // extern "C"

namespace {
// The evaluation criterion's pipeline (§3.3): row DFT, column DFT + power + Parseval sums
// per sigma, fixed-order reductions.  Error images from the counts of `level` (img == nullptr) or
// given on the device (img [ni][P], the smooth family).
int eval_pipeline(bn_ctx* ctx, uint32_t level, uint32_t ni, const double* img, const double* sigmas, uint32_t ns,
                  double* rmse, double* spectrum, double* profile) {
    const uint32_t L = ctx->L, P = ctx->P;
    const uint8_t* rows = img ? nullptr : u8_rows(ctx);
    if (!img) {
        CUDA_TRY(ctx->iref.ensure(ctx->Ts));
        k_iref<<<(ctx->Ts + 127) / 128, 128, 0, ctx->stream>>>(ctx->ab.p, ctx->pxy.p, ctx->Ts, ctx->iref.p);
        LAUNCHED();
    }
    // twiddles w^m = exp(-2 pi i m / L) and the 1D kernel spectra h_s(k) = sum_d g(d) cos(2 pi k d / L) / sum_d g(d)
    // (g = exp(-d^2 / (2 sigma^2)), |d| <= ceil(4 sigma)): host libm, like the energy tables
    const double two_pi = 6.283185307179586476925286766559;
    std::vector<double2> tw(L);
    for (uint32_t m = 0; m < L; ++m) tw[m] = make_double2(std::cos(two_pi * m / L), -std::sin(two_pi * m / L));
    const uint32_t nsk = ns ? ns : 1;
    std::vector<double> h((size_t)nsk * L, 0.0);
    for (uint32_t s = 0; s < ns; ++s) {
        const int r = (int)std::ceil(4.0 * sigmas[s]);
        double Z = 0.0;
        for (int d = -r; d <= r; ++d) Z += std::exp(-(double)d * d / (2.0 * sigmas[s] * sigmas[s]));
        for (uint32_t k = 0; k < L; ++k) {
            double acc = 0.0;
            for (int d = -r; d <= r; ++d)
                acc += std::exp(-(double)d * d / (2.0 * sigmas[s] * sigmas[s])) *
                       std::cos(two_pi * (double)(((int64_t)k * d % (int64_t)L + L) % L) / L);
            h[(size_t)s * L + k] = acc / Z;
        }
    }
    const uint32_t chunk = 1024, ngroups = (ni + EV_II - 1) / EV_II;
    CUDA_TRY(ctx->ev_tw.ensure(L));
    CUDA_TRY(ctx->ev_h.ensure(h.size()));
    CUDA_TRY(ctx->ev_X1.ensure((size_t)std::min(chunk, ni) * P));
    CUDA_TRY(ctx->ev_rm.ensure((size_t)ni * L * nsk));
    CUDA_TRY(ctx->ev_sp.ensure((size_t)ngroups * P));
    CUDA_TRY(ctx->ev_out.ensure(64 + P + L / 2));
    CUDA_TRY(cudaMemcpyAsync(ctx->ev_tw.p, tw.data(), L * sizeof(double2), cudaMemcpyHostToDevice, ctx->stream));
    CUDA_TRY(cudaMemcpyAsync(ctx->ev_h.p, h.data(), h.size() * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
    const size_t sm1 = (size_t)L * EV_II * 8 + L * 16, sm2 = (size_t)L * EV_II * 16 + L * 16 + (size_t)L * EV_II * 8;
    CUDA_TRY(cudaFuncSetAttribute(k_ev_dft_rows, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm1));
    CUDA_TRY(cudaFuncSetAttribute(k_ev_dft_cols, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm2));
    const double invN = 1.0 / (double)ctx->levels[level];
    for (uint32_t i0 = 0; i0 < ni; i0 += chunk) {
        const uint32_t ci = std::min(chunk, ni - i0);
        const dim3 grid(L, (ci + EV_II - 1) / EV_II);
        k_ev_dft_rows<<<grid, 256, sm1, ctx->stream>>>(rows, L, ctx->rowB, level * ctx->Tp, invN, ctx->iref.p, i0,
                                                        ci, ctx->ev_tw.p, ctx->ev_X1.p, img);
        LAUNCHED();
        k_ev_dft_cols<<<grid, 256, sm2, ctx->stream>>>(ctx->ev_X1.p, L, i0, ci, ctx->ev_tw.p, ctx->ev_h.p, nsk,
                                                        ctx->ev_rm.p, ctx->ev_sp.p);
        LAUNCHED();
    }
    double* dr = ctx->ev_out.p;
    double* dS = dr + 64;
    double* dprof = dS + P;
    if (ns) {
        k_ev_rmse<<<ns, 256, 0, ctx->stream>>>(ctx->ev_rm.p, L, ni, nsk, dr);
        LAUNCHED();
        CUDA_TRY(cudaMemcpyAsync(rmse, dr, ns * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    }
    if (spectrum || profile) {
        k_ev_spectrum<<<1, 256, 0, ctx->stream>>>(ctx->ev_sp.p, L, ngroups, ni, dS, dprof);
        LAUNCHED();
        if (spectrum) CUDA_TRY(cudaMemcpyAsync(spectrum, dS, (size_t)P * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
        if (profile)
            CUDA_TRY(cudaMemcpyAsync(profile, dprof, (L / 2) * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    }
    CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    return BN_OK;
}

int check_eval_args(bn_ctx* ctx, uint32_t level, const double* sigmas, uint32_t ns, const double* rmse) {
    int rc;
    if ((rc = check_ready(ctx))) return rc;
    if (level >= ctx->nl) return fail(ctx, BN_EINVAL, "level %u >= %u levels", level, ctx->nl);
    if (ns > 64 || (ns && (!sigmas || !rmse))) return fail(ctx, BN_EINVAL, "bad sigma list (at most 64)");
    for (uint32_t s = 0; s < ns; ++s)
        if (!(sigmas[s] > 0) || !std::isfinite(sigmas[s]) || sigmas[s] > 1e4)
            return fail(ctx, BN_EINVAL, "sigma[%u] = %g outside (0, 1e4]", s, sigmas[s]);
    if (ctx->L > 256) return fail(ctx, BN_EINVAL, "the evaluation criterion supports L <= 256 (L = %u)", ctx->L);
    return BN_OK;
}
}  // namespace

extern "C" {

int bn_eval_quality(bn_ctx* ctx, uint32_t level, const double* sigmas, uint32_t ns, double* rmse, double* spectrum,
                    double* profile) {
    if (!ctx) return BN_EINVAL;
    int rc;
    if ((rc = check_eval_args(ctx, level, sigmas, ns, rmse))) return rc;
    DeviceGuard g(ctx->dev);
    if ((rc = ensure_counts(ctx))) return rc;
    return eval_pipeline(ctx, level, ctx->Ts, nullptr, sigmas, ns, rmse, spectrum, profile);
}

int bn_eval_smooth(bn_ctx* ctx, uint32_t level, uint32_t n_bumps, const double* bumps, const double* sigmas,
                   uint32_t ns, double* rmse, double* spectrum, double* profile, double* iref) {
    if (!ctx) return BN_EINVAL;
    int rc;
    if ((rc = check_eval_args(ctx, level, sigmas, ns, rmse))) return rc;
    if (n_bumps == 0 || !bumps) return fail(ctx, BN_EINVAL, "empty bump list");
    std::vector<double> ref(n_bumps);
    const double r2 = 1.4142135623730950488016887242097, sqrt_half_pi = 1.2533141373155002512078826424055;
    for (uint32_t i = 0; i < n_bumps; ++i) {
        const double cx = bumps[4 * i], cy = bumps[4 * i + 1], sx = bumps[4 * i + 2], sy = bumps[4 * i + 3];
        if (!(sx > 0) || !(sy > 0) || !std::isfinite(sx) || !std::isfinite(sy) || !std::isfinite(cx) || !std::isfinite(cy))
            return fail(ctx, BN_EINVAL, "bump %u: widths must be positive and finite", i);
        // exact reference: separable erf product over [0,1]^2 (host libm)
        ref[i] = sx * sqrt_half_pi * (std::erf((1.0 - cx) / (sx * r2)) + std::erf(cx / (sx * r2))) *
                 (sy * sqrt_half_pi * (std::erf((1.0 - cy) / (sy * r2)) + std::erf(cy / (sy * r2))));
    }
    if (iref) memcpy(iref, ref.data(), n_bumps * sizeof(double));
    DeviceGuard g(ctx->dev);
    const uint32_t P = ctx->P;
    CUDA_TRY(ctx->ev_bump.ensure((size_t)n_bumps * 5));
    CUDA_TRY(ctx->ev_img.ensure((size_t)n_bumps * P));
    double* dref = ctx->ev_bump.p + 4 * (size_t)n_bumps;
    CUDA_TRY(cudaMemcpyAsync(ctx->ev_bump.p, bumps, (size_t)n_bumps * 4 * sizeof(double), cudaMemcpyHostToDevice,
                             ctx->stream));
    CUDA_TRY(cudaMemcpyAsync(dref, ref.data(), n_bumps * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
    const size_t n = (size_t)n_bumps * P;
    k_ev_smooth_err<<<(unsigned)((n + 255) / 256), 256, 0, ctx->stream>>>(
        ctx->U.p, ctx->S.p, ctx->levels[level], reinterpret_cast<const double4*>(ctx->ev_bump.p), dref, n_bumps, P,
        ctx->ev_img.p);
    LAUNCHED();
    return eval_pipeline(ctx, level, n_bumps, ctx->ev_img.p, sigmas, ns, rmse, spectrum, profile);
}

int bn_set_permutation(bn_ctx* ctx, const uint32_t* perm, uint32_t n) {
    if (!ctx) return BN_EINVAL;
    if (!perm || n == 0) return fail(ctx, BN_EINVAL, "empty permutation");
    std::vector<uint8_t> seen(n, 0);
    for (uint32_t j = 0; j < n; ++j) {
        if (perm[j] >= n || seen[perm[j]])
            return fail(ctx, BN_EINVAL, "not a permutation of [0, %u): entry %u = %u", n, j, perm[j]);
        seen[perm[j]] = 1;
    }
    DeviceGuard g(ctx->dev);
    std::vector<uint32_t> inv(n);
    for (uint32_t j = 0; j < n; ++j) inv[perm[j]] = j;
    CUDA_TRY(ctx->perm.ensure(n));
    CUDA_TRY(ctx->invperm.ensure(n));
    CUDA_TRY(cudaMemcpyAsync(ctx->perm.p, perm, (size_t)n * sizeof(uint32_t), cudaMemcpyHostToDevice, ctx->stream));
    CUDA_TRY(cudaMemcpyAsync(ctx->invperm.p, inv.data(), (size_t)n * sizeof(uint32_t), cudaMemcpyHostToDevice, ctx->stream));
    CUDA_TRY(cudaStreamSynchronize(ctx->stream));  // the caller's array and `inv` may go away
    ctx->perm_n = n;
    return BN_OK;
}

int bn_window_distances(bn_ctx* ctx, int32_t* out, int is_device) {
    if (!ctx) return BN_EINVAL;
    if (!out) return fail(ctx, BN_EINVAL, "null output");
    DeviceGuard g(ctx->dev);
    int rc = ensure_work(ctx);
    if (rc) return rc;
    if ((rc = gram_only(ctx))) return rc;
    const size_t n = (size_t)ctx->nl * ctx->P * half_count(ctx->R);
    int* dst = out;
    DevBuf<int> tmp;
    if (!is_device) {
        CUDA_TRY(tmp.ensure(n));
        dst = tmp.p;
    }
    k_dt_export<<<(unsigned)((n + 255) / 256), 256, 0, ctx->stream>>>(ctx->Dt.p, ctx->P, ctx->nl, ctx->R, dst);
    LAUNCHED();
    if (!is_device) {
        cudaError_t e = cudaMemcpyAsync(out, dst, n * sizeof(int), cudaMemcpyDeviceToHost, ctx->stream);
        if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
        tmp.release();
        if (e != cudaSuccess) return fail(ctx, BN_ECUDA, "distances readback: %s", cudaGetErrorString(e));
    }
    return BN_OK;
}

int bn_profile_enable(bn_ctx* ctx, int enable) {
    if (!ctx) return BN_EINVAL;
    DeviceGuard g(ctx->dev);
    flush_profile(ctx);
    if (enable)
        for (int i = 0; i < BN_K_COUNT_IDS; ++i) ctx->prof_ms[i] = 0.0, ctx->prof_n[i] = 0;
    ctx->prof = enable != 0;
    return BN_OK;
}

int bn_profile_get(bn_ctx* ctx, uint32_t kernel_id, double* total_ms, uint64_t* launches) {
    if (!ctx) return BN_EINVAL;
    if (kernel_id >= BN_K_COUNT_IDS) return fail(ctx, BN_EINVAL, "kernel id %u", kernel_id);
    DeviceGuard g(ctx->dev);
    flush_profile(ctx);
    if (total_ms) *total_ms = ctx->prof_ms[kernel_id];
    if (launches) *launches = ctx->prof_n[kernel_id];
    return BN_OK;
}

int bn_comm_unique_id(void* out128) {
    if (!out128) return BN_EINVAL;
    if (!g_nccl.load()) return BN_ENCCL;
    NcclUid id;
    if (g_nccl.get_uid(&id)) return BN_ENCCL;
    memcpy(out128, &id, sizeof id);
    return BN_OK;
}

int bn_comm_init(bn_ctx* ctx, const void* uid, int rank, int world) {
    if (!ctx) return BN_EINVAL;
    if (!uid || world < 1 || rank < 0 || rank >= world) return fail(ctx, BN_EINVAL, "bad rank/world");
    if (!g_nccl.load()) return fail(ctx, BN_ENCCL, "libnccl.so.2 not loadable: %s", dlerror());
    DeviceGuard g(ctx->dev);
    NcclUid id;
    memcpy(&id, uid, sizeof id);
    NcclComm comm = nullptr;
    int r = g_nccl.init_rank(&comm, world, id, rank);
    if (r) return fail(ctx, BN_ENCCL, "ncclCommInitRank: %s", g_nccl.errstr(r));
    if (ctx->comm) g_nccl.destroy(ctx->comm);
    ctx->comm = comm;
    ctx->rank = rank;
    ctx->world = world;
    return BN_OK;
}

}  // extern "C"
