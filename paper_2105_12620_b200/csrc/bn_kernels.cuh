// bn_kernels.cuh -- sm_100a kernels of the blue-noise sampler optimiser hot path.
//
// Pass structure.  Within a pass every pixel p receives exactly ONE candidate
// row cn_p (REDRAW: counts of a Philox-drawn shift; SWAP: the partner's row), and the 64 colour
// classes are visited in order.  Hence, at any moment of the pass, pixel q is in one of two
// states, c_q (not yet accepted) or cn_q (accepted earlier in this pass), and every energy
// change the pass can need is a function of the four window distances
//     D(c_p,c_q), D(cn_p,c_q), D(c_p,cn_q), D(cn_p,cn_q)          (q = p + o, o in the window).
// The pass therefore runs as
//   k_counts / k_swap_gather : candidate rows cn (+ norms)                      [ALU]
//   k_gram                   : the four windowed distances for every (p, o in H)  [dominant]
//   k_lut                    : per (p, o): delta0 = q(D(cn_p,c_q)) - q(D(c_p,c_q)),
//                              delta1 = q(D(cn_p,cn_q)) - q(D(c_p,cn_q)) (int128, summed over
//                              levels), and E of the pass-start state
//   k_decide (x64 classes)   : dE_p = 2 * sum_o (accepted[q] ? delta1 : delta0); accept iff < 0
//   k_commit, k_pass_stats   : copy accepted rows / shifts; exact per-pass sums
// which is bit-identical to the step-by-step greedy algorithm (oracle) because distances are
// exact integers and the fixed-point energy terms are summed exactly in int128.
//
// H = half window {o : oy > 0 or (oy == 0 and ox > 0)}: each unordered neighbour pair is
// computed once and written to both (p, o) and (p + o, -o).
#pragma once
#include <cuda.h>  // CUtensorMap (type only; the encoder is fetched through the runtime)
#include <cstdint>
#include <cuda_runtime.h>

namespace bn {

// Debug build (-DBN_DEBUG_BOUNDS, tools/gpu_debug.sh): device bounds checks at the index
// computations of the pass kernels; a failed check traps (the launch fails with an error).
#ifdef BN_DEBUG_BOUNDS
#define BN_ASSERT(c)          \
    do {                      \
        if (!(c)) __trap();   \
    } while (0)
#else
#define BN_ASSERT(c) \
    do {             \
    } while (0)
#endif

typedef __int128 i128;
typedef unsigned __int128 u128;

// ------------------------------------------------------------------------------ Philox4x32-10
// Salmon et al. SC'11.  Written independently of the oracle; parity checked via accept logs.
__device__ __forceinline__ uint4 philox4x32_10(uint4 c, uint2 k) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        if (r) {
            k.x += 0x9E3779B9u;
            k.y += 0xBB67AE85u;
        }
        const uint32_t lo0 = 0xD2511F53u * c.x, hi0 = __umulhi(0xD2511F53u, c.x);
        const uint32_t lo1 = 0xCD9E8D57u * c.z, hi1 = __umulhi(0xCD9E8D57u, c.z);
        c = make_uint4(hi1 ^ c.y ^ k.x, lo1, hi0 ^ c.w ^ k.y, lo0);
    }
    return c;
}
__device__ __forceinline__ uint4 philox_seeded(uint64_t seed, uint32_t c0, uint32_t c1, uint32_t c2,
                                               uint32_t c3) {
    return philox4x32_10(make_uint4(c0, c1, c2, c3), make_uint2((uint32_t)seed, (uint32_t)(seed >> 32)));
}

// Pixel of active index m in colour class s = 8r + k of pass t (stride-8 staggered schedule).
__device__ __forceinline__ uint32_t class_pixel(uint32_t L, uint64_t seed, uint32_t t, uint32_t s, uint32_t m) {
    const uint32_t nb = L >> 3, b = m / nb, a = m - b * nb, r = s >> 3, k = s & 7;
    const uint32_t delta = philox_seeded(seed, b, t, r, 2).x;
    const uint32_t along = 8 * a + ((delta + k) & 7), across = 8 * b + r;
    return (t & 1) ? along * L + across : across * L + along;
}
__device__ __forceinline__ uint32_t swap_kappa(uint64_t seed, uint32_t t, uint32_t s, uint32_t M) {
    return 1u + philox_seeded(seed, s, t, 0, 3).x % (M - 1u);
}
// SWAP partner of pixel p in pass t: invert class_pixel (class s = 8r + k, active index m), then
// the pixel of m ^ kappa(t, s) in the same class.
__device__ __forceinline__ uint32_t swap_partner(uint32_t L, uint64_t seed, uint32_t t, uint32_t p) {
    const uint32_t nb = L >> 3, M = nb * nb, x = p & (L - 1), y = p / L;
    const uint32_t along = (t & 1) ? y : x, across = (t & 1) ? x : y;
    const uint32_t r = across & 7, b = across >> 3;
    const uint32_t delta = philox_seeded(seed, b, t, r, 2).x & 7;
    const uint32_t s = 8 * r + ((along - delta) & 7), m = b * nb + (along >> 3);
    return class_pixel(L, seed, t, s, m ^ swap_kappa(seed, t, s, M));
}
// Same as class_pixel with delta(t, r, b) & 7 read from a per-pass table tab[r * nb + b].
__device__ __forceinline__ uint32_t class_pixel_tab(const uint8_t* tab, uint32_t L, uint32_t t, uint32_t s,
                                                    uint32_t m) {
    const uint32_t nb = L >> 3, b = m / nb, a = m - b * nb, r = s >> 3, k = s & 7;
    const uint32_t along = 8 * a + ((tab[r * nb + b] + k) & 7), across = 8 * b + r;
    return (t & 1) ? along * L + across : across * L + along;
}

// Window indexing.  Full window W: raster over (oy, ox) in [-R,R]^2 minus the centre.
__host__ __device__ __forceinline__ int win_index(int ox, int oy, int R) {
    const int w = (oy + R) * (2 * R + 1) + (ox + R), centre = R * (2 * R + 1) + R;
    return w > centre ? w - 1 : w;
}
// Half window H: oy = 0, ox = 1..R first, then oy = 1..R, ox = -R..R.
__host__ __device__ __forceinline__ int half_index(int ox, int oy, int R) {
    return oy == 0 ? ox - 1 : R + (oy - 1) * (2 * R + 1) + (ox + R);
}
// Padded half window (the layout of the window-distance planes): row oy = 0 holds ox = 1..R in
// ru4(R) records, rows oy = 1..R hold ox = -R..R in ru4(2R+1) records each, so every window row of
// a pixel starts 32-byte aligned in an int2 plane and a Gram epilogue writes it with whole-sector
// stores.  Pad records are never read.
__host__ __device__ constexpr int ru4(int x) { return (x + 3) & ~3; }
__host__ __device__ constexpr int half_count_padded(int R) { return ru4(R) + R * ru4(2 * R + 1); }
__host__ __device__ __forceinline__ int hpad_index(int ox, int oy, int R) {
    return oy == 0 ? ox - 1 : ru4(R) + (oy - 1) * ru4(2 * R + 1) + (ox + R);
}

// ---------------------------------------------------------------------------- narrow row formats
// Row formats of a level's count rows (SURVEY §8 f3 narrow storage): see the Gram.
enum : uint32_t { BN_FMT_U8 = 0, BN_FMT_E2M1 = 1, BN_FMT_E3M2 = 2 };
__host__ __device__ constexpr uint32_t fmt_bits(uint32_t f) { return f == BN_FMT_U8 ? 8 : f == BN_FMT_E2M1 ? 4 : 6; }
// Codes (the encoders are byte-parallel, in pack_chunk16): e2m1 |d| <= 4: 0 1 2 3 4 -> 0x0 0x2 0x4 0x5
// 0x6, sign 0x8; e3m2 |d| <= 8: (1 + mantissa/4) 2^(e-3): 0 1 2 3 4 5 6 7 8 -> 0x00 0x0C 0x10 0x12
// 0x14 0x15 0x16 0x17 0x18, sign 0x20.
__device__ __forceinline__ int dec_e2m1(uint32_t c) {
    const uint32_t m = c & 7u;
    const int a = m == 0 ? 0 : m == 2 ? 1 : m == 4 ? 2 : m == 5 ? 3 : 4;
    return (c & 8u) ? -a : a;
}
__device__ __forceinline__ int dec_e3m2(uint32_t c) {
    const uint32_t e = (c >> 2) & 7u, mt = c & 3u;
    const int a = e == 0 ? 0 : (int)((4u + mt) << e) >> 5;  // 2^(e-3) (1 + mt/4) for e >= 3
    return (c & 0x20u) ? -a : a;
}
// Row layout of a level: byte offset lb[l] in the row, format fmt[l].  One warp per pixel row;
// lane j packs the 16-integrand groups j, j + 32, ...: e2m1 16 x 4 bit in 8 bytes, e3m2 16 x 6 bit
// in 12 bytes (element k at bit bits * k of its group, little-endian), u8 copied; norms |delta|^2
// (|c|^2 for u8 levels) per level.
struct NarrowLayout {
    uint32_t fmt[8], lb[8];
};
// Pack one 16-integrand chunk of a level row (16 counts cv, offsets ov) in format f at group g of
// the level's packed row dst; adds sum delta^2 (sum c^2 for u8) to nrm, returns max |delta| (u8: 0).
__device__ __forceinline__ uint32_t pack_chunk16(uint4 cv, uint4 ov, uint32_t f, uint8_t* dst, uint32_t g, int& nrm) {
    const uint32_t cw[4] = {cv.x, cv.y, cv.z, cv.w}, ow[4] = {ov.x, ov.y, ov.z, ov.w};
    if (f == BN_FMT_U8) {
        reinterpret_cast<uint4*>(dst)[g] = cv;
#pragma unroll
        for (int k = 0; k < 4; ++k) nrm = (int)__dp4a(cw[k], cw[k], (unsigned)nrm);
        return 0;
    }
    uint32_t mx = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) mx = __vmaxu4(mx, __vabsdiffu4(cw[k], ow[k]));
    mx = max(max(mx & 0xffu, (mx >> 8) & 0xffu), max((mx >> 16) & 0xffu, mx >> 24));
    if (f == BN_FMT_E2M1) {  // byte-parallel; |d| <= 4 where the format is valid (range checked)
        uint32_t w[2] = {0, 0};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const uint32_t ad = __vabsdiffu4(cw[k], ow[k]);  // |d| per byte
            // e2m1 code per byte: magnitude a + min(a, 2) (0 1 2 3 4 -> 0 2 4 5 6), sign 0x8
            const uint32_t code = (ad + __vminu4(ad, 0x02020202u)) | (__vcmpltu4(cw[k], ow[k]) & 0x08080808u);
            nrm = (int)__dp4a(ad, ad, (unsigned)nrm);
            const uint32_t t = code | (code >> 4);  // byte 0 = n0 | n1 << 4, byte 2 = n2 | n3 << 4
            w[k >> 1] |= __byte_perm(t, 0, 0x4420) << (16 * (k & 1));
        }
        reinterpret_cast<uint2*>(dst)[g] = make_uint2(w[0], w[1]);
    } else {  // e3m2, byte-parallel; |d| <= 8 where the format is valid (range checked)
        uint32_t v[4];  // four 24-bit runs of four 6-bit codes
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const uint32_t ad = __vabsdiffu4(cw[k], ow[k]);  // |d| per byte, 0..8
            nrm = (int)__dp4a(ad, ad, (unsigned)nrm);
            const uint32_t t = ad | (ad >> 4);
            const uint32_t sel = __byte_perm(t, 0, 0x4420);  // selector nibbles |d0| .. |d3| (mod 8)
            // codes of 0..7: 00 0C 10 12 | 14 15 16 17; |d| = 8: 0x18; sign 0x20
            const uint32_t eq8 = __vcmpeq4(ad, 0x08080808u);
            uint32_t code = (__byte_perm(0x12100C00u, 0x17161514u, sel) & ~eq8) | (0x18181818u & eq8);
            code |= __vcmpltu4(cw[k], ow[k]) & 0x20202020u;
            v[k] = (code & 0x3Fu) | ((code >> 2) & 0xFC0u) | ((code >> 4) & 0x3F000u) | ((code >> 6) & 0xFC0000u);
        }
        uint32_t* d32 = reinterpret_cast<uint32_t*>(dst + 12 * g);  // element j at bits 6j .. 6j+5
        d32[0] = v[0] | (v[1] << 24);
        d32[1] = (v[1] >> 8) | (v[2] << 16);
        d32[2] = (v[2] >> 16) | (v[3] << 8);
    }
    return mx;
}

// ---------------------------------------------------------------------------- error vectors
// Heaviside counts for every pixel of a tile (set_tile) or for the REDRAW candidates of pass t.
//   c_l,p,i = #{k < N_l : a_i (X_k - PX_i) + b_i (Y_k - PY_i) >= 0},  X_k = S_k.x + u_p.x mod 2^32.
// With X' = X - 2^31 as int32, the test is a_i X' + b_i Y' >= C_i,  C_i = a PX + b PY - (a+b) 2^31,
// i.e. two 32x32->64 integer multiply-adds per (pixel, integrand, sample): exact.
// Padding integrands (i >= Ts) use a = b = 0, C = 2^62, so they always count 0 (t = -C).
// Layout out: [p][l][Tp] uint8; norms: [p][l] int32 = sum_i c^2.
#ifndef BN_COUNT_PIX
#define BN_COUNT_PIX 8
#endif
constexpr int COUNT_PIX = BN_COUNT_PIX;  // pixels per CTA (short CTAs co-schedule well on the aux stream)

// Filtered fast test.  t = fma(a, x', fma(b, y', -C)) in fp32 with x' = fl(X'), C~ = fl(C):
//   |x' - X'| <= 2^6, |C~ - C| <= 2^24, |a|,|b| <= 2^15, |b y' - C~| < 2^49
//   => |t - v| <= 2^21 + 2^24 + 2^21 + 2^24 + 2^25 < 2^27
// so sign(t) = sign(v) whenever |t| >= 2^27.  A (pixel, integrand) whose samples ever come
// closer than that (probability ~2^-20 per test) is recounted exactly in int64.
constexpr float COUNT_EXACT_BAND = 134217728.0f;  // 2^27

// Packed fp32x2 FMA (sm_100: FFMA2), round-to-nearest on each half exactly like fmaf.
__device__ __forceinline__ unsigned long long fma2(unsigned long long a, unsigned long long b, unsigned long long c) {
    unsigned long long d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
    return d;
}
__device__ __forceinline__ unsigned long long pack2(float lo, float hi) {
    return (unsigned long long)__float_as_uint(lo) | ((unsigned long long)__float_as_uint(hi) << 32);
}

// Sign counting of a pair of integrands (2h, 2h+1) in ONE u32.  PRMT with the sign-replicating
// selector 0xFFBB turns the packed results (t_lo, t_hi) into S_lo * 0x0000FFFF + S_hi * 0xFFFF0000
// (S = sign bit of t = 1 for a negative test); subtracting it from the accumulator gives
//   acc = n_lo + 2^16 (n_hi - n_lo)  (mod 2^32),  n = number of negative tests so far (< 2^15),
// from which both counts are recovered exactly (sign_counts).  Two samples share one IADD3:
// 0.75 ALU-pipe instructions per test instead of 1.25 (LEA.HI / SHF + IADD3).
__device__ __forceinline__ uint32_t sgn2(unsigned long long t) {
    uint32_t d;
    asm("prmt.b32 %0, %1, %2, 0xFFBB;" : "=r"(d) : "r"((uint32_t)t), "r"((uint32_t)(t >> 32)));
    return d;
}
__device__ __forceinline__ void sign_counts(uint32_t acc, uint32_t& n_lo, uint32_t& n_hi) {
    n_lo = acc & 0xffffu;
    n_hi = n_lo + (uint32_t)((int)(acc - n_lo) >> 16);
}
__device__ __forceinline__ float min_abs2(float m, unsigned long long t) {
    return fminf(m, fminf(fabsf(__uint_as_float((uint32_t)t)), fabsf(__uint_as_float((uint32_t)(t >> 32)))));  // FMNMX3
}

// Samples k (and k+1) against NI integrands held as NI/2 packed pairs: t = a x + (b y - C) per lane half.
template <int NI>
__device__ __forceinline__ void count_sample2(float2 p0, float2 p1, const unsigned long long* ab2a,
                                              const unsigned long long* ab2b, const unsigned long long* c2,
                                              uint32_t* acc, float* mn) {
    const unsigned long long xx0 = pack2(p0.x, p0.x), yy0 = pack2(p0.y, p0.y);
    const unsigned long long xx1 = pack2(p1.x, p1.x), yy1 = pack2(p1.y, p1.y);
#pragma unroll
    for (int h = 0; h < NI / 2; ++h) {
        const unsigned long long t0 = fma2(ab2a[h], xx0, fma2(ab2b[h], yy0, c2[h]));
        const unsigned long long t1 = fma2(ab2a[h], xx1, fma2(ab2b[h], yy1, c2[h]));
        acc[h] = acc[h] - sgn2(t0) - sgn2(t1);  // IADD3
        mn[h] = min_abs2(min_abs2(mn[h], t0), t1);
    }
}
template <int NI>
__device__ __forceinline__ void count_sample1(float2 p0, const unsigned long long* ab2a, const unsigned long long* ab2b,
                                              const unsigned long long* c2, uint32_t* acc, float* mn) {
    const unsigned long long xx0 = pack2(p0.x, p0.x), yy0 = pack2(p0.y, p0.y);
#pragma unroll
    for (int h = 0; h < NI / 2; ++h) {
        const unsigned long long t0 = fma2(ab2a[h], xx0, fma2(ab2b[h], yy0, c2[h]));
        acc[h] -= sgn2(t0);
        mn[h] = min_abs2(mn[h], t0);
    }
}

// Samples [k0, k1) of NPX pixels at once (independent accumulator chains: more ILP per warp).
template <int NI, int NPX>
__device__ __forceinline__ void count_span(const float2* const* xyf, uint32_t k0, uint32_t k1,
                                           const unsigned long long* a2, const unsigned long long* b2,
                                           const unsigned long long* c2, uint32_t (*acc)[NI / 2],
                                           float (*mn)[NI / 2]) {
    uint32_t k = k0;
    constexpr uint32_t STEP = NPX == 1 ? 4 : 2;
    for (; k + STEP <= k1; k += STEP) {
#pragma unroll
        for (int x = 0; x < NPX; ++x) {
            count_sample2<NI>(xyf[x][k], xyf[x][k + 1], a2, b2, c2, acc[x], mn[x]);
            if (NPX == 1) count_sample2<NI>(xyf[x][k + 2], xyf[x][k + 3], a2, b2, c2, acc[x], mn[x]);
        }
    }
    for (; k + 2 <= k1; k += 2)
#pragma unroll
        for (int x = 0; x < NPX; ++x) count_sample2<NI>(xyf[x][k], xyf[x][k + 1], a2, b2, c2, acc[x], mn[x]);
    if (k < k1)
#pragma unroll
        for (int x = 0; x < NPX; ++x) count_sample1<NI>(xyf[x][k], a2, b2, c2, acc[x], mn[x]);
}

// Each thread owns NI = 8 consecutive integrands (two packed 32-bit words per level row) and
// walks the CTA's pixels; the sample loop is split at the level boundaries N_l so that the
// inner loop is branch-free and unrolled.  The fp32 operands of the filtered test come
// pre-packed from k_count_prep (one 96-byte record per integrand group).
constexpr int COUNT_NI = 8;
struct CountGroup {  // integrand pairs (2h, 2h+1) of one group, h = 0..3: {a, a}, {b, b}, {-C, -C}
    unsigned long long a2[COUNT_NI / 2], b2[COUNT_NI / 2], c2[COUNT_NI / 2];
};
__global__ void k_count_prep(const int2* __restrict__ ab, const long long* __restrict__ Cc, uint32_t Tp,
                             CountGroup* __restrict__ g) {
    const uint32_t q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= Tp / COUNT_NI) return;
    CountGroup r;
#pragma unroll
    for (int h = 0; h < COUNT_NI / 2; ++h) {
        const int2 v0 = ab[COUNT_NI * q + 2 * h], v1 = ab[COUNT_NI * q + 2 * h + 1];
        r.a2[h] = pack2((float)v0.x, (float)v1.x);
        r.b2[h] = pack2((float)v0.y, (float)v1.y);
        r.c2[h] = pack2(-__ll2float_rn(Cc[COUNT_NI * q + 2 * h]), -__ll2float_rn(Cc[COUNT_NI * q + 2 * h + 1]));
    }
    g[q] = r;
}

// NPX pixels (pp, pp + nsub, ...) of the CTA against integrand group q: counts per level, row
// norms, and the warp-cooperative exact recount of ambiguous pairs (see k_counts).
template <int NI, int NPX>
__device__ __forceinline__ void count_pixels(uint32_t pp0, uint32_t nsub, uint32_t p0, const CountGroup& gq, uint32_t q,
                                             const float2* sXYf, const int2* sXY, uint32_t ns, const uint32_t* levels,
                                             uint32_t nl, uint32_t Tp, uint32_t Nmax, uint8_t* __restrict__ out,
                                             const int2* __restrict__ ab, const long long* __restrict__ Cc,
                                             int (*sNorm)[8]) {
    const uint32_t lane = threadIdx.x & 31;
    uint32_t acc[NPX][NI / 2];  // packed negative-test counts per pair of integrands (sgn2)
    float mn[NPX][NI / 2];      // min |t| per pair of integrands
    const float2* xyf[NPX];
#pragma unroll
    for (int x = 0; x < NPX; ++x) {
        xyf[x] = sXYf + (pp0 + x * nsub) * ns;
#pragma unroll
        for (int j = 0; j < NI / 2; ++j) acc[x][j] = 0, mn[x][j] = 3.0e38f;
    }
    uint32_t kprev = 0;
    for (uint32_t li = 0; li < nl; ++li) {
        const uint32_t n1 = levels[li];
        count_span<NI, NPX>(xyf, kprev, n1, gq.a2, gq.b2, gq.c2, acc, mn);
        kprev = n1;
#pragma unroll
        for (int x = 0; x < NPX; ++x) {
            const uint32_t pp = pp0 + x * nsub;
            uint32_t neg[NI];
#pragma unroll
            for (int h = 0; h < NI / 2; ++h) sign_counts(acc[x][h], neg[2 * h], neg[2 * h + 1]);
            uint32_t w[NI / 4];
            uint32_t nsq = 0;
#pragma unroll
            for (int h = 0; h < NI / 4; ++h) {
                const uint32_t c0 = n1 - neg[4 * h], c1 = n1 - neg[4 * h + 1];
                const uint32_t c2 = n1 - neg[4 * h + 2], c3 = n1 - neg[4 * h + 3];
                w[h] = c0 | (c1 << 8) | (c2 << 16) | (c3 << 24);
                nsq = __dp4a(w[h], w[h], nsq);  // sum of the four squared counts
            }
            uint8_t* orow = out + (size_t)(p0 + pp) * nl * Tp + NI * q;
            *reinterpret_cast<uint2*>(orow + (size_t)li * Tp) = make_uint2(w[0], w[1]);
            // a warp's lanes share the pixel (q runs over whole warps): one REDUX, one atomic
            nsq = __reduce_add_sync(0xffffffffu, nsq);
            if (lane == 0) atomicAdd(&sNorm[pp][li], (int)nsq);
        }
    }
    // exact int64 recount of any pair of integrands whose samples came within the error band,
    // done by the whole warp (the pixel is warp-uniform): lane k tests samples k, k+32, ...;
    // per-level counts are popcounts of the ballots
#pragma unroll
    for (int x = 0; x < NPX; ++x) {
        const uint32_t pp = pp0 + x * nsub;
        uint8_t* orow = out + (size_t)(p0 + pp) * nl * Tp + NI * q;
#pragma unroll
        for (int h = 0; h < NI / 2; ++h) {
            uint32_t need = __ballot_sync(0xffffffffu, mn[x][h] < COUNT_EXACT_BAND);
            while (need) {
                const int src = __ffs(need) - 1;
                need &= need - 1;
                const uint32_t qs = __shfl_sync(0xffffffffu, q, src);
                for (int e = 0; e < 2; ++e) {
                    const uint32_t i = NI * qs + 2 * h + e;
                    const int2 abj = ab[i];
                    const long long cj = Cc[i];
                    uint32_t bits[4];
#pragma unroll
                    for (int r = 0; r < 4; ++r) {
                        const uint32_t k = lane + 32 * r;
                        bool pos = false;
                        if (k < Nmax) {
                            const int2 xy = sXY[pp * ns + k];
                            pos = ((long long)abj.x * xy.x + (long long)abj.y * xy.y - cj) >= 0;
                        }
                        bits[r] = __ballot_sync(0xffffffffu, pos);
                    }
                    if ((int)lane == src) {
                        for (uint32_t lj = 0; lj < nl; ++lj) {
                            const uint32_t n1 = levels[lj];
                            uint32_t cnt = 0;
#pragma unroll
                            for (int r = 0; r < 4; ++r) {
                                const uint32_t lo = 32 * r;
                                const uint32_t m = n1 <= lo ? 0u : n1 - lo >= 32 ? 0xffffffffu : (1u << (n1 - lo)) - 1u;
                                cnt += __popc(bits[r] & m);
                            }
                            uint8_t* cell = orow + (size_t)lj * Tp + 2 * h + e;
                            const int old = *cell;
                            *cell = (uint8_t)cnt;
                            atomicAdd(&sNorm[pp][lj], (int)(cnt * cnt) - old * old);
                        }
                    }
                }
            }
        }
    }
}

// <= 120 registers: a counts CTA (8 warps) then fits beside a persistent Gram CTA (10 warps x 104)
// in one SM's 64 K registers, so another tile's counts overlap the Gram (the e2e serving loop)
#ifndef BN_COUNT_MAXREG
#define BN_COUNT_MAXREG 120
#endif
__global__ void __maxnreg__(BN_COUNT_MAXREG) k_counts(const uint2* __restrict__ U, uint2* __restrict__ Uout, int redraw,
                                                uint64_t seed, uint32_t pass_t, uint32_t P,
                                                const int2* __restrict__ ab, const long long* __restrict__ Cc,
                                                const CountGroup* __restrict__ grp, uint32_t Tp,
                                                const uint2* __restrict__ S, uint32_t Nmax, uint4 lev_lo,
                                                uint4 lev_hi, uint32_t nl, uint8_t* __restrict__ out,
                                                int* __restrict__ norms, unsigned int* __restrict__ rows_done,
                                                uint32_t L) {
    constexpr int NI = COUNT_NI;
    // the CTA's samples, [COUNT_PIX][ns] each (dynamic, ns = Nmax rounded up to 4: a small footprint
    // lets a counts CTA of another tile co-reside with a persistent Gram CTA on the same SM)
    extern __shared__ __align__(16) uint8_t kc_smem[];
    const uint32_t ns = (Nmax + 3) & ~3u;
    float2* sXYf = reinterpret_cast<float2*>(kc_smem);
    int2* sXY = reinterpret_cast<int2*>(sXYf + COUNT_PIX * ns);
    __shared__ int sNorm[COUNT_PIX][8];
    __shared__ uint32_t levels[8];
    if (threadIdx.x == 0) {
        levels[0] = lev_lo.x, levels[1] = lev_lo.y, levels[2] = lev_lo.z, levels[3] = lev_lo.w;
        levels[4] = lev_hi.x, levels[5] = lev_hi.y, levels[6] = lev_hi.z, levels[7] = lev_hi.w;
    }
    const uint32_t p0 = blockIdx.x * COUNT_PIX;
    // threads = (integrand group q) x (pixel subset sub): when Tp/NI < blockDim the CTA's threads
    // split its pixels instead of idling (Tp/NI is a multiple of 32, so warps stay uniform)
    const uint32_t qn = Tp / NI;
    const uint32_t nsub = qn < blockDim.x ? blockDim.x / qn : 1;
    const uint32_t sub = threadIdx.x / (blockDim.x / nsub), tq = threadIdx.x % (blockDim.x / nsub);
    // this thread's first integrand group: loads in flight while the samples are staged
    CountGroup g0;
    if (tq < qn) g0 = grp[tq];
    for (uint32_t j = threadIdx.x; j < COUNT_PIX * 8; j += blockDim.x) (&sNorm[0][0])[j] = 0;
    // samples X_k = S_k + u_p: warp w stages pixels w, w + 8, ...; every lane of the warp draws
    // the pixel's shift (one Philox per pixel and lane) instead of waiting behind a barrier
    for (uint32_t pp = threadIdx.x >> 5; pp < COUNT_PIX; pp += blockDim.x >> 5) {
        const uint32_t p = p0 + pp;
        if (p >= P) break;
        uint2 u;
        if (redraw) {  // candidate j = redraw - 1 (best-of-K draws j = 0 .. K-1)
            const uint4 r = philox_seeded(seed, p, pass_t, (uint32_t)(redraw - 1), 1);
            u = make_uint2(r.x, r.y);
            if ((threadIdx.x & 31) == 0) Uout[p] = u;
        } else {
            u = U[p];
        }
        for (uint32_t k = threadIdx.x & 31; k < Nmax; k += 32) {
            const uint2 sk = S[k];
            const int2 xy = make_int2((int)((sk.x + u.x) ^ 0x80000000u), (int)((sk.y + u.y) ^ 0x80000000u));
            sXY[pp * ns + k] = xy;
            sXYf[pp * ns + k] = make_float2(__int2float_rn(xy.x), __int2float_rn(xy.y));
        }
    }
    __syncthreads();
    const uint32_t lane = threadIdx.x & 31;
    for (uint32_t q = tq; q < qn; q += blockDim.x / nsub) {
        const CountGroup gq = q == tq ? g0 : grp[q];
        for (uint32_t pp = sub; pp < COUNT_PIX; pp += 2 * nsub) {
            if (p0 + pp >= P) break;
            if (pp + nsub < COUNT_PIX && p0 + pp + nsub < P)  // two of the thread's pixels at once
                count_pixels<NI, 2>(pp, nsub, p0, gq, q, sXYf, sXY, ns, levels, nl, Tp, Nmax, out, ab, Cc, sNorm);
            else
                count_pixels<NI, 1>(pp, nsub, p0, gq, q, sXYf, sXY, ns, levels, nl, Tp, Nmax, out, ab, Cc, sNorm);
        }
    }
    __syncthreads();
    for (uint32_t j = threadIdx.x; j < COUNT_PIX * nl; j += blockDim.x) {
        const uint32_t pp = j / nl, l = j - pp * nl;
        if (p0 + pp < P) norms[(size_t)(p0 + pp) * nl + l] = sNorm[pp][l];
    }
    if (rows_done) {  // publish: this CTA's segment of tile row p0 / L is complete (rows, norms, shifts)
        __threadfence();
        __syncthreads();
        if (threadIdx.x == 0) atomicAdd(rows_done + p0 / L, 1u);
    }
}
// Tp / 8 integrand groups per pixel: callers guarantee Tp % 256 == 0 (whole warps per group).

// SWAP partner map of pass t: part[p] = p2 for every couple member (one thread per (class, index);
// 3 Philox draws per thread instead of per copying thread).  The rows are then gathered by
// k_paper_gather (one warp per pixel, 16-byte copies).
__global__ void k_swap_pairs(uint32_t L, uint64_t seed, uint32_t pass_t, uint32_t* __restrict__ part) {
    const uint32_t M = (L / 8) * (L / 8);
    const uint32_t sm = blockIdx.x * blockDim.x + threadIdx.x;  // s * M + m
    if (sm >= 64 * M) return;
    const uint32_t s = sm / M, m = sm - s * M;
    const uint32_t kappa = swap_kappa(seed, pass_t, s, M);
    part[class_pixel(L, seed, pass_t, s, m)] = class_pixel(L, seed, pass_t, s, m ^ kappa);
}

// ------------------------------------------------------------------- window-distance planes
// The window distances of every (level l, pixel p, half-window offset h) are two int2 planes over
// the same [l][p][h] index (the int4 buffer Dt of nl*P*H records holds plane 0 in its first half,
// plane 1 in its second):  plane 0 = (D(c_p, c_q), D(c_p, cn_q)),  plane 1 = (D(cn_p, c_q),
// D(cn_p, cn_q)).  A Gram epilogue owning the c_p (or cn_p) row of a pixel writes whole int2
// records of one plane, so its stores coalesce.
__host__ __device__ __forceinline__ int2* dt_plane(int4* Dt, size_t n, int v) {
    return reinterpret_cast<int2*>(Dt) + (size_t)v * n;
}
__device__ __forceinline__ void dt_put(int4* Dt, size_t n, size_t idx, int4 d) {
    dt_plane(Dt, n, 0)[idx] = make_int2(d.x, d.y);
    dt_plane(Dt, n, 1)[idx] = make_int2(d.z, d.w);
}
#ifndef BN_DT_LDCS
#define BN_DT_LDCS 1  // C3 decide 0.0695 -> 0.066 ms: the dE tables written by k_lut stay in L2
#endif
__device__ __forceinline__ int4 dt_get(const int4* Dt, size_t n, size_t idx) {
    if (BN_DT_LDCS) {  // streaming loads: read once, keep the freshly written dE tables in L2 instead
        const int2 a = __ldcs(reinterpret_cast<const int2*>(Dt) + idx), b = __ldcs(reinterpret_cast<const int2*>(Dt) + n + idx);
        return make_int4(a.x, a.y, b.x, b.y);
    }
    const int2 a = __ldg(reinterpret_cast<const int2*>(Dt) + idx), b = __ldg(reinterpret_cast<const int2*>(Dt) + n + idx);
    return make_int4(a.x, a.y, b.x, b.y);
}

__device__ __forceinline__ void cp_async16(uint32_t smem, const void* gmem) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem), "l"(gmem) : "memory");
}

// ------------------------------------------------- window Gram on 5th-gen tensor cores (tcgen05)
// tcgen05 helpers: shared-memory matrix descriptors (K-major, 128-B swizzle), instruction
// descriptors, MMA issue / commit, mbarrier waits and TMEM loads.
namespace tc {
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr) {  // K-major, SWIZZLE_128B, SBO = 1024
    return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) |
           ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}
__host__ __device__ constexpr uint32_t idesc_u8(int M, int N) {
    return (2u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);  // s32 += u8 x u8, K-major
}
__device__ __forceinline__ void mma(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc, uint32_t accum) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(da), "l"(db), "r"(idesc), "r"(accum));
}
__device__ __forceinline__ void commit(uint32_t bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ bool mbar_try(uint32_t bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred P;\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2;\n\tselp.u32 %0, 1, 0, P;\n\t}"
        : "=r"(ok)
        : "r"(bar), "r"(parity)
        : "memory");
    return ok;
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
    for (uint32_t i = 0; !mbar_try(bar, parity); ++i)
        if (i > (1u << 26)) __trap();  // never hang the GPU on a protocol bug
}
__device__ __forceinline__ void ld8(uint32_t taddr, uint32_t* r) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "r"(taddr));
}
__device__ __forceinline__ void ld32(uint32_t taddr, uint32_t* r) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
          "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
          "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
          "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
}
}  // namespace tc

__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void named_bar(int id, int n) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

// TMA-fed, warp-specialised tcgen05 window Gram, one (8x8 block, level) item at a time.
// Every operand group is an aligned run of 8 pixels (x0 is a multiple of 8), i.e. 8 consecutive
// rows of the [y][x][row] count tensor: one TMA box of 8 rows x 128 elements per group, which is
// exactly one SWIZZLE_128B atom of the UMMA K-major layout.  Per 128-element K stage: A = the c and
// cn rows of the 64 block pixels (M = 128), B = the c and cn rows of 5 neighbour rows x 3 aligned
// groups covering x0-8 .. x0+15 (N = 240; the 2 columns outside the window are ignored).  A toroidal
// wrap only ever moves a whole group.  Warps 0-3: epilogue, warp 4 lane 0: TMA producer, warp 5
// lane 0: UMMA issuer.  Three neighbour chunks (the R = 7 geometry, a superset of every R <= 7),
// two TMEM accumulators of 256 columns.
namespace tc3 {
constexpr int R = 7, NBR = 8 + R, GRP = 3, NBX = 8 * GRP /*24*/;
constexpr int CH_ROWS = 5, NCHUNK = 3, N = 2 * CH_ROWS * NBX /*240*/;
constexpr int A_BYTES = 128 * 128, B_BYTES = N * 128;
constexpr int STAGE = A_BYTES + B_BYTES;  // 47104 = 46 KB
#ifndef BN_GRAM_NSTAGE
#define BN_GRAM_NSTAGE 4
#endif
constexpr int NSTAGE = BN_GRAM_NSTAGE;
// warps 0-7: two epilogue groups (group g drains TMEM accumulator g, i.e. every other neighbour
// chunk; warp & 3 = its TMEM lane quadrant), warp 8: TMA producer, warp 9: MMA issuer
#ifndef BN_GRAM_EPI_GROUPS
#define BN_GRAM_EPI_GROUPS 2
#endif
constexpr int EPI = BN_GRAM_EPI_GROUPS;  // epilogue groups of 4 warps (1 or 2)
constexpr int THREADS = 32 * (4 * EPI + 2);
constexpr int SCR = 25;  // odd row stride: conflict-free scratch writes
constexpr int SMEM = NSTAGE * STAGE + EPI * (4 * 32 * SCR * 4 + 2 * NBR * NBX * 4) + 1024;
constexpr int H = 2 * R * R + 2 * R;
}  // namespace tc3

__device__ __forceinline__ void tma_2d(uint32_t dst, const CUtensorMap* map, int x, int y, uint32_t bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
            dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(bar)
        : "memory");
}

__device__ __forceinline__ void tma_3d(uint32_t dst, const CUtensorMap* map, int x, int y, int z, uint32_t bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
            dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(z), "r"(bar)
        : "memory");
}
// Tensor maps over the [y][x][K] count tensor (3D, K innermost): box A = {128, 8, 8} (a whole
// 8x8 block = 64 rows), box B = {128, 24, 5} (a whole neighbour chunk, no wrap), box S =
// {128, 8, 1} (8 pixels of one row, used where a toroidal wrap splits a chunk).
// Per level and operand: a = the block's A rows {128, 8 px, 8 rows}; b = a whole neighbour chunk
// {128, 24 px, 5 rows}; g = one 8-pixel group of a chunk {128, 8, 5} (x-wrapping chunks, group-major
// in shared memory); r = one chunk row {128, 24, 1} (y-wrapping chunks); s = {128, 8, 1} (corners).
struct CountMaps {
    CUtensorMap a, b, s, g, r;
};

// 256-bit store of four int2 records {(x[0], y[0]) .. (x[3], y[3])} (one whole 32-byte sector).
__device__ __forceinline__ void st_v8(int2* dst, const int* x, const int* y) {
    asm volatile("st.global.v8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(dst), "r"(x[0]), "r"(y[0]), "r"(x[1]),
                 "r"(y[1]), "r"(x[2]), "r"(y[2]), "r"(x[3]), "r"(y[3])
                 : "memory");
}

// -------------------------------------------------------------------------- energy terms
// q(o, D) = rn_u64(2^52 * W[o] * G_l[D]); W and G are host-built fp64 tables (exp/sqrt of the
// host libm), the product is one IEEE multiply (no contraction possible), the scaling by 2^52
// is exact (reading R15).  With q < 2^52, every dE term (a sum over <= 8 levels of differences of
// two q's) satisfies |term| < 2^55, and every window sum of <= 224 terms |sum| < 2^63: int64 is
// exact throughout the decisions.
constexpr int BN_FIX_BITS = 52;  // E = E_fixed * 2^-52
__device__ __forceinline__ unsigned long long qterm(double w, const double* __restrict__ G, int D) {
    return __double2ull_rn(__dmul_rn(__dmul_rn(w, __ldg(G + D)), 4503599627370496.0));
}

// dE terms are int64 (exact, see above).  The int128 escape machinery of earlier versions (a
// sentinel plus a side table for terms beyond int64) is unreachable with the 2^52 scale; the
// invariant |term| < 2^55 is checked here (err flag 2).
constexpr long long DT_ESC = (long long)0x8000000000000000ull;
constexpr long long TERM_MAX = 1ll << 55;
__device__ __forceinline__ void put_terms(longlong2* d, size_t idx, long long v0, long long v1, int* err) {
    if (v0 >= TERM_MAX || v0 <= -TERM_MAX || v1 >= TERM_MAX || v1 <= -TERM_MAX) atomicOr(err, 2);
    d[idx] = make_longlong2(v0, v1);
}
__device__ __forceinline__ i128 get_term(long long v, const longlong2* __restrict__ x, size_t idx) {
    if (v != DT_ESC) return (i128)v;
    const longlong2 e = x[idx];
    return ((i128)e.y << 64) | (u128)(unsigned long long)e.x;
}
struct DTabs {
    const longlong2* d;  // {delta0, delta1} interleaved per (pixel, offset): one 16-B access per term
    const longlong2* x0;
    const longlong2* x1;
};

// Exact warp sum of an int128 (two's complement, mod 2^128) with 8 REDUX.SUM instructions:
// split into 16-bit limbs (each warp sum < 2^21 fits 32 bits), then recombine with carries.
__device__ __forceinline__ i128 warp_sum_i128_redux(unsigned long long lo, unsigned long long hi) {
    uint32_t s[8];
#pragma unroll
    for (int i = 0; i < 4; ++i) s[i] = __reduce_add_sync(0xffffffffu, (uint32_t)(lo >> (16 * i)) & 0xffffu);
#pragma unroll
    for (int i = 0; i < 4; ++i) s[4 + i] = __reduce_add_sync(0xffffffffu, (uint32_t)(hi >> (16 * i)) & 0xffffu);
    u128 r = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) r += (u128)s[i] << (16 * i);
    return (i128)r;
}

// Exact warp sum of a u128 (or an int128 mod 2^128) by a 5-step shuffle butterfly.
__device__ __forceinline__ u128 warp_sum_u128(u128 v) {
    unsigned long long lo = (unsigned long long)v, hi = (unsigned long long)(v >> 64);
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        const unsigned long long olo = __shfl_xor_sync(0xffffffffu, lo, o);
        const unsigned long long ohi = __shfl_xor_sync(0xffffffffu, hi, o);
        const unsigned long long nlo = lo + olo;
        hi += ohi + (nlo < lo);
        lo = nlo;
    }
    return ((u128)hi << 64) | lo;
}

// Exact warp sum of int64 partials whose total fits int64: four independent REDUX.SUM over 16-bit
// limbs of the two's-complement value (each limb sum < 2^21), recombined mod 2^64.
#ifndef BN_I64_REDUX
#define BN_I64_REDUX 1  // 0: 5-step shuffle butterfly (C3 decide 0.073 vs 0.070 ms, C2 0.068 vs 0.058)
#endif
__device__ __forceinline__ long long warp_sum_i64(long long v) {
    if (BN_I64_REDUX) {
        const unsigned long long u = (unsigned long long)v;
        unsigned long long r = 0;
#pragma unroll
        for (int i = 0; i < 4; ++i)
            r += (unsigned long long)__reduce_add_sync(0xffffffffu, (uint32_t)(u >> (16 * i)) & 0xffffu) << (16 * i);
        return (long long)r;
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

struct LutArgs {
    const double* G[8];  // per-level G tables
    int Dmax[8];         // largest legal D per level (guards corrupted distances)
};

// NL > 0: compile-time level count (all distance loads issued up front); NL = 0: runtime nl.
template <int R, int NL>
__global__ void __launch_bounds__(256) k_lut(const int4* __restrict__ Dt, uint32_t L, uint32_t nl_rt,
                                             const double* __restrict__ W, LutArgs lut, int write_deltas,
                                             longlong2* __restrict__ d, u128* __restrict__ Epart, int* __restrict__ err) {
    constexpr int HP = half_count_padded(R), R0 = ru4(R), RW = ru4(2 * R + 1);
    constexpr int WN = (2 * R + 1) * (2 * R + 1) - 1;
    const uint32_t P = L * L;
#ifndef BN_LUT_REVERSE
#define BN_LUT_REVERSE 1
#endif
    // (p, padded offset hp); BN_LUT_REVERSE: last-written window distances first (still in L2)
    const size_t idx = BN_LUT_REVERSE ? (size_t)(gridDim.x - 1 - blockIdx.x) * blockDim.x + threadIdx.x
                                      : (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    unsigned long long e = 0;  // < 2 * 8 * 2^52 = 2^56 per thread, < 2^61 per warp
    const uint32_t p = (uint32_t)(idx / HP), hp = (uint32_t)(idx - (size_t)p * HP);
    int ox, oy;
    if (hp < (uint32_t)R0) {
        oy = 0;
        ox = (int)hp + 1;
    } else {
        oy = 1 + (int)(hp - R0) / RW;
        ox = (int)(hp - R0) % RW - R;
    }
    if (idx < (size_t)P * HP && ox <= R) {  // pads (ox > R) are skipped
        const uint32_t x = p % L, y = p / L;
        const uint32_t q = ((y + oy) & (L - 1)) * L + ((x + ox + L) & (L - 1));
        const int wi = win_index(ox, oy, R), wm = win_index(-ox, -oy, R);
        BN_ASSERT(p < P && q < P && wi >= 0 && wi < WN && wm >= 0 && wm < WN);
        const double w = W[wi];
        // q < 2^52: per-level differences and their sums over <= 8 levels are exact in int64 (R15)
        long long a0 = 0, a1 = 0, b0 = 0, b1 = 0;
        const uint32_t nl = NL ? NL : nl_rt;
        int4 Dv[NL ? NL : 1];
        if (NL) {
#pragma unroll
            for (int l = 0; l < (NL ? NL : 1); ++l) Dv[l] = dt_get(Dt, (size_t)nl * P * HP, (size_t)l * P * HP + idx);
        }
#pragma unroll
        for (uint32_t l = 0; l < nl; ++l) {
            const int4 D = NL ? Dv[NL ? l : 0] : dt_get(Dt, (size_t)nl * P * HP, (size_t)l * P * HP + idx);
            const int dm = lut.Dmax[l];
            if ((unsigned)D.x > (unsigned)dm || (unsigned)D.y > (unsigned)dm || (unsigned)D.z > (unsigned)dm ||
                (unsigned)D.w > (unsigned)dm) {
                atomicOr(err, 1);
                continue;
            }
            const double* G = lut.G[l];
            const long long qcc = (long long)qterm(w, G, D.x), qcn = (long long)qterm(w, G, D.y);
            const long long qnc = (long long)qterm(w, G, D.z), qnn = (long long)qterm(w, G, D.w);
            e += (unsigned long long)qcc;
            a0 += qnc - qcc;  // p takes cn_p, q still c_q
            a1 += qnn - qcn;  // p takes cn_p, q already cn_q
            b0 += qcn - qcc;  // q takes cn_q, p still c_p
            b1 += qnn - qnc;  // q takes cn_q, p already cn_p
        }
        e *= 2;  // ordered pairs (p,q) and (q,p)
        if (write_deltas) {
            put_terms(d, (size_t)p * WN + wi, a0, a1, err);
            put_terms(d, (size_t)q * WN + wm, b0, b1, err);
        }
    }
    // block reduction of e: exact warp sums of 16-bit limbs (REDUX), then the 8 warp partials
    __shared__ unsigned long long swarp[8];
    unsigned long long ws = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i)
        ws += (unsigned long long)__reduce_add_sync(0xffffffffu, (uint32_t)(e >> (16 * i)) & 0xffffu) << (16 * i);
    if ((threadIdx.x & 31) == 0) swarp[threadIdx.x >> 5] = ws;
    __syncthreads();
    if (threadIdx.x == 0) {
        u128 t = 0;
        for (int j = 0; j < (int)(blockDim.x >> 5); ++j) t += swarp[j];
        Epart[blockIdx.x] = t;
    }
}

// Row formats of a level's count rows (SURVEY §8 f3 narrow storage).  BN_FMT_U8:
// the counts c (uint8, kind::i8, exact s32 accumulation).  BN_FMT_E2M1 / BN_FMT_E3M2: the deltas
// delta = c - off_i (off_i = round(N_l I_ref,i), one integer per integrand and level) packed 16 per
// 8 (e2m1, 4-bit, |delta| <= 4 exact) or 12 bytes (e3m2, 6-bit, |delta| <= 8 exact); the TMA
// unpacks them into the same 128-B-swizzled shared-memory layout as bytes and the tensor core
// multiplies them with kind::f8f6f4 into fp32 (exact: |<x,y>| < 2^24; tools/narrow_mma_check.cu).
// The offsets cancel in every distance: D = sum (c_p - c_q)^2 = sum (delta_p - delta_q)^2, and the
// norms stored beside the rows are |delta|^2.
__host__ __device__ constexpr uint32_t idesc_f8(uint32_t f, int M, int N) {  // f32 += e2m1 / e3m2, K-major
    return (1u << 4) | ((f == BN_FMT_E2M1 ? 5u : 4u) << 7) | ((f == BN_FMT_E2M1 ? 5u : 4u) << 10) |
           ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
// e2m1 rows left packed (two values per byte, 256 per 128-B row) for kind::mxf4 (block32, every
// ue8m0 scale factor 2^0 = 0x7F, so the products are the plain integer products; exact fp32 sums,
// tools/narrow_mma_check.cu): K = 64 per instruction, twice the f8f6f4 rate and half the TMA rows.
__host__ __device__ constexpr uint32_t idesc_mxf4(int M, int N) {
    return (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | (1u << 23) | ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ void mma_mxf4(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc, uint32_t accum,
                                         uint32_t tmem_sf) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], %1, %2, %3, [%5], [%5], p;\n\t}" ::"r"(tmem_d),
        "l"(da), "l"(db), "r"(idesc), "r"(accum), "r"(tmem_sf));
}
// K elements per 128-B row of a stage: packed e2m1 (mxf4) holds 256
__host__ __device__ constexpr uint32_t stage_k(uint32_t f) { return f == BN_FMT_E2M1 ? 256 : 128; }
__device__ __forceinline__ void mma_f8(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc, uint32_t accum) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f8f6f4 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(da), "l"(db), "r"(idesc), "r"(accum));
}
// TMA maps of every level (c and cn operands) and the level's row format.
struct GramMaps {
    CountMaps c[8], n[8];
    uint32_t fmt[8];
};

// Persistent window Gram: one CTA per SM walks the (8x8 block, level) items cta, cta + G, ...
// The stage ring and the two TMEM accumulators continue across items, so the TMA producer and
// the MMA warp run into the next item while the epilogue still drains the previous one, and the
// per-CTA start-up (TMEM allocation, barrier set-up) is paid once per SM.  The epilogue loads the
// next item's neighbourhood norms itself after finishing an item (its MMAs are already running),
// forms D = |x|^2 + |y|^2 - 2<x,y> for the half-window offsets of radius R and writes each
// (pixel, window row) run of the two int2 planes with whole-sector 256-bit stores.
template <int R>
__global__ void __launch_bounds__(tc3::THREADS, 1) k_gram_tc4(const __grid_constant__ GramMaps gm,
                                                              const int* __restrict__ nc, const int* __restrict__ nn,
                                                              uint32_t L, uint32_t Tp, uint32_t nl,
                                                              int4* __restrict__ Dt,
                                                              const unsigned int* __restrict__ rows_done,
                                                              uint32_t rows_target,
                                                              const uint32_t* __restrict__ border,
                                                              unsigned int* __restrict__ sched, uint32_t csplit) {
    using tc3::NBR; using tc3::NBX; using tc3::GRP; using tc3::CH_ROWS; using tc3::NCHUNK; using tc3::N;
    using tc3::A_BYTES; using tc3::STAGE; using tc3::NSTAGE; using tc3::SCR;
    constexpr int RW = ru4(2 * R + 1), R0 = ru4(R), NV = RW > R + 1 + R0 ? RW : R + 1 + R0;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    const uint32_t raw = (uint32_t)__cvta_generic_to_shared(smem_raw);
    const uint32_t sring = (raw + 1023) & ~1023u;
    uint8_t* gring = smem_raw + (sring - raw);
    int* scratch = reinterpret_cast<int*>(gring + NSTAGE * STAGE);  // [2 groups][4 warps][32][SCR]
    int* snorm_all = scratch + tc3::EPI * 4 * 32 * SCR;                // [groups][2][NBR][NBX], x from x0-8
    constexpr int IQ = 4;  // item ring (dynamic scheduling): producer -> MMA warp and epilogue
    __shared__ __align__(8) uint64_t bars[2 * NSTAGE + 4 + 2 * IQ];
    __shared__ uint32_t tmem_sh, sItem[IQ];
    const uint32_t b_full = (uint32_t)__cvta_generic_to_shared(&bars[0]);
    const uint32_t b_empty = b_full + 8 * NSTAGE, b_tfull = b_full + 16 * NSTAGE, b_tempty = b_tfull + 16;
    const uint32_t i_full = b_tempty + 16, i_empty = i_full + 8 * IQ;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // csplit = NCHUNK (small tiles: fewer (block, level) pairs than SMs): an item is one neighbour
    // chunk of a (block, level), so three CTAs share a block instead of one walking its chunks
    const uint32_t nbx = L / 8, nitems = nbx * nbx * nl * csplit, P = L * L;
    constexpr uint32_t SF_COL = 240;  // scale factors (mxf4) in the unused columns 240..247 of accumulator 0
    if (threadIdx.x == 0) {
        for (int i = 0; i < NSTAGE; ++i) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b_full + 8 * i) : "memory");
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b_empty + 8 * i) : "memory");
        }
        for (int i = 0; i < 2; ++i) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b_tfull + 8 * i) : "memory");
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 128;" ::"r"(b_tempty + 8 * i) : "memory");
        }
        for (int i = 0; i < IQ; ++i) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(i_full + 8 * i) : "memory");
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(i_empty + 8 * i), "r"(1 + tc3::EPI) : "memory");
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                         (uint32_t)__cvta_generic_to_shared(&tmem_sh))
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = tmem_sh;
    if (warp < 4) {  // ue8m0 scale factors 2^0 for the mxf4 levels (all 128 lanes, 8 columns)
        asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1};" ::"r"(
                         tmem + ((uint32_t)(32 * warp) << 16) + SF_COL), "r"(0x7F7F7F7Fu) : "memory");
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    // Items block-major (the levels of a block consecutive) so that the window distances written last
    // are whole pixels' rows, which k_lut (BN_LUT_REVERSE) reads first while they are still in L2.
    // Block order `border` (host-built): the blocks whose chunks wrap the torus (more, smaller TMA
    // boxes: the slowest items) first, so the static round-robin spreads them over the CTAs.
    auto item_xyl = [&](uint32_t it, uint32_t& x0, uint32_t& y0, uint32_t& l) {
        it /= csplit;
        l = it % nl;
        const uint32_t b = border ? (uint32_t)border[it / nl] : it / nl;
        x0 = 8 * (b % nbx);
        y0 = 8 * (b / nbx);
    };
    // the item's chunks [ch0, ch1)
    auto item_ch = [&](uint32_t it, int& ch0, int& ch1) {
        ch0 = csplit == 1 ? 0 : (int)(it % csplit);
        ch1 = csplit == 1 ? NCHUNK : ch0 + 1;
    };
    // wait until every tile row y0 .. y0 + 14 (mod L) of this pass's candidates is published by
    // k_counts (acquire), then order the following TMA (async-proxy) reads after it
    auto wait_rows = [&](uint32_t y0) {
        if (!rows_done) return;
        for (uint32_t r = 0; r < (uint32_t)NBR; ++r) {
            const unsigned int* f = rows_done + ((y0 + r) & (L - 1));
            for (uint32_t n = 0;; ++n) {
                unsigned int v;
                asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(f) : "memory");
                if ((int)(v - rows_target) >= 0) break;
                if (n > (1u << 26)) __trap();  // never hang the GPU on a protocol bug
                __nanosleep(64);
            }
        }
        asm volatile("fence.proxy.async.global;" ::: "memory");
    };

    // Dynamic scheduling (sched != null): the producer claims the next item from the global counter
    // sched[0] and hands it to the MMA warp and the epilogue through the ring sItem (slot full /
    // empty mbarriers; the empty barrier collects the MMA warp's and the epilogue's release), so a CTA
    // that drew slow (wrapping) items simply takes fewer; the last CTA resets the counters.  Static
    // round robin (it = cta, cta + G, ...) otherwise.
    auto next_item = [&](uint32_t j, uint32_t prev) -> uint32_t {  // j-th item of this CTA (consumer side)
        if (!sched) return j == 0 ? blockIdx.x : prev + gridDim.x;
        const uint32_t slot = j % IQ;
        tc::mbar_wait(i_full + 8 * slot, (j / IQ) & 1);
        return sItem[slot];
    };
    auto release_item = [&](uint32_t j) {
        if (sched) mbar_arrive(i_empty + 8 * (j % IQ));
    };
    if (warp == 4 * tc3::EPI) {
        // --------------------------------------------------------------- TMA producer
        if (lane == 0) {
            uint32_t g = 0, j = 0;
            for (uint32_t it = blockIdx.x;; ++j) {
                if (sched) {
                    const uint32_t slot = j % IQ;
                    if (j >= (uint32_t)IQ) tc::mbar_wait(i_empty + 8 * slot, ((j / IQ) - 1) & 1);
                    it = atomicAdd(sched, 1u);
                    sItem[slot] = it;
                    mbar_arrive(i_full + 8 * slot);  // release (CTA scope): sItem written first
                } else if (j > 0) {
                    it += gridDim.x;
                }
                if (it >= nitems) break;
                uint32_t x0, y0, l;
                item_xyl(it, x0, y0, l);
                int chb, che;
                item_ch(it, chb, che);
                wait_rows(y0);
                // transaction bytes = the packed global bytes the boxes read (128 + 240 rows)
                const uint32_t f = gm.fmt[l], nk = Tp / stage_k(f);
                const uint32_t tx = (uint32_t)(128 + N) * 128 * (f == BN_FMT_E2M1 ? 8 : fmt_bits(f)) / 8;
                for (int ch = chb; ch < che; ++ch)
                    for (uint32_t ks = 0; ks < nk; ++ks, ++g) {
                        const uint32_t b = g % NSTAGE, use = g / NSTAGE;
                        if (use > 0) tc::mbar_wait(b_empty + 8 * b, (use - 1) & 1);
                        const uint32_t buf = sring + b * STAGE, bar = b_full + 8 * b;
#ifdef BN_GRAM_PROBE_NOTMA  // timing probe (not product): no operand loads
                        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
                        continue;
#endif
                        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(tx)
                                     : "memory");
                        const int kx = (int)(ks * 128);
#ifdef BN_GRAM_PROBE_WHOLE  // timing probe (not product): wrapping chunks as one (zero-filled) box
                        const bool xw = false, yw = false;
#else
                        const bool xw = x0 < 8 || x0 + 16 > L, yw = y0 + CH_ROWS * (ch + 1) > L;
#endif
                        for (int v = 0; v < 2; ++v) {
                            const CountMaps& m = v ? gm.n[l] : gm.c[l];
                            tma_3d(buf + v * 8192, &m.a, kx, (int)x0, (int)y0, bar);  // 64 block rows
                            const uint32_t bdst = buf + A_BYTES + v * CH_ROWS * GRP * 1024;
                            if (!xw && !yw) {
                                tma_3d(bdst, &m.b, kx, (int)x0 - 8, (int)(y0 + CH_ROWS * ch), bar);
                            } else if (!yw) {  // x wrap: three 8-pixel groups, group-major [gx][row][px]
                                for (int gx = 0; gx < GRP; ++gx)
                                    tma_3d(bdst + gx * CH_ROWS * 1024, &m.g, kx, (int)((x0 + 8 * gx + L - 8) & (L - 1)),
                                           (int)(y0 + CH_ROWS * ch), bar);
                            } else if (!xw) {  // y wrap: five rows of 24 pixels
                                for (int nyl = 0; nyl < CH_ROWS; ++nyl)
                                    tma_3d(bdst + nyl * GRP * 1024, &m.r, kx, (int)x0 - 8,
                                           (int)((y0 + CH_ROWS * ch + nyl) & (L - 1)), bar);
                            } else {
                                for (int nyl = 0; nyl < CH_ROWS; ++nyl)
                                    for (int gx = 0; gx < GRP; ++gx) {
                                        const uint32_t py = (y0 + CH_ROWS * ch + nyl) & (L - 1);
                                        const uint32_t px = (x0 + 8 * gx + L - 8) & (L - 1);
                                        tma_3d(bdst + (nyl * GRP + gx) * 1024, &m.s, kx, (int)px, (int)py, bar);
                                    }
                            }
                        }
                    }
            }
        }
    } else if (warp == 4 * tc3::EPI + 1) {
        // --------------------------------------------------------------- UMMA issuer
        uint32_t g = 0, cc = 0;  // stage counter, chunk counter (accumulator ring)
        for (uint32_t ji = 0, it = 0;; ++ji) {
            it = next_item(ji, it);
            __syncwarp();
            if (lane == 0) release_item(ji);
            if (it >= nitems) break;
            uint32_t x0, y0, l;
            item_xyl(it, x0, y0, l);
            const uint32_t f = gm.fmt[l], nk = Tp / stage_k(f);
            const uint32_t idesc = f == BN_FMT_U8 ? tc::idesc_u8(128, N) : f == BN_FMT_E2M1 ? idesc_mxf4(128, N) : idesc_f8(f, 128, N);
            int chb, che;
            item_ch(it, chb, che);
            for (int ch = chb; ch < che; ++ch, ++cc) {
                const uint32_t ub = cc & 1, uu = cc >> 1;
                if (uu > 0) tc::mbar_wait(b_tempty + 8 * ub, (uu - 1) & 1);
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                for (uint32_t ks = 0; ks < nk; ++ks, ++g) {
                    const uint32_t b = g % NSTAGE;
                    tc::mbar_wait(b_full + 8 * b, (g / NSTAGE) & 1);
                    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                    if (lane == 0) {
                        const uint32_t sa = sring + b * STAGE, sb = sa + A_BYTES;
#ifndef BN_GRAM_PROBE_NOMMA
#pragma unroll
                        for (int kk = 0; kk < 4; ++kk) {
                            if (f == BN_FMT_U8)
                                tc::mma(tmem + 256 * ub, tc::sdesc(sa + 32 * kk), tc::sdesc(sb + 32 * kk), idesc,
                                        (ks > 0 || kk > 0) ? 1u : 0u);
                            else if (f == BN_FMT_E2M1)
                                mma_mxf4(tmem + 256 * ub, tc::sdesc(sa + 32 * kk), tc::sdesc(sb + 32 * kk), idesc,
                                         (ks > 0 || kk > 0) ? 1u : 0u, tmem + SF_COL);
                            else
                                mma_f8(tmem + 256 * ub, tc::sdesc(sa + 32 * kk), tc::sdesc(sb + 32 * kk), idesc,
                                       (ks > 0 || kk > 0) ? 1u : 0u);
                        }
#endif
                        tc::commit(b_empty + 8 * b);
                        if (ks + 1 == nk) tc::commit(b_tfull + 8 * ub);
                    }
                    __syncwarp();
                }
            }
        }
    } else if (warp < 4 * tc3::EPI) {
        // --------------------------------------------------------------- epilogue (2 groups)
        const int grp = warp >> 2, wq = warp & 3, tg = threadIdx.x & 127, gbar = 2 + grp;
        const int arow = 32 * wq + lane, v = arow >> 6, pp = arow & 63, dy = pp >> 3, dx = pp & 7;
        int* scr = scratch + ((grp * 4 + wq) * 32 + lane) * SCR;
        int* snorm = snorm_all + grp * 2 * NBR * NBX;
        uint32_t cc = 0;
        for (uint32_t ji = 0, it = 0;; ++ji) {
            it = next_item(ji, it);
            named_bar(gbar, 128);  // every thread of the group read the slot (and the previous item's norms are done)
            if (tg == 0) release_item(ji);
            if (it >= nitems) break;
            uint32_t x0, y0, l;
            item_xyl(it, x0, y0, l);
            const bool fp = gm.fmt[l] != BN_FMT_U8;  // fp32 accumulator (exact integers)
            if (tg == 0) wait_rows(y0);  // the candidates' norms come from k_counts too
            named_bar(gbar, 128);
            for (int j = tg; j < 2 * NBR * NBX; j += 128) {
                const int nx = j % NBX, vr = j / NBX, vv = vr >= NBR, r = vr - vv * NBR;
                const uint32_t qy = (y0 + r) & (L - 1), qx = (x0 + nx + L - 8) & (L - 1);
                snorm[j] = (vv ? nn : nc)[(size_t)(qy * L + qx) * nl + l];
            }
            named_bar(gbar, 128);
            const uint32_t p = ((y0 + dy) & (L - 1)) * L + ((x0 + dx) & (L - 1));
            BN_ASSERT(p < P && l < nl);
            const int np = snorm[(v * NBR + dy) * NBX + dx + 8];
            int2* out2 = dt_plane(Dt, (size_t)nl * P * half_count_padded(R), v) + ((size_t)l * P + p) * half_count_padded(R);
            int chb, che;
            item_ch(it, chb, che);
            for (int ch = chb; ch < che; ++ch, ++cc) {
                const uint32_t ub = cc & 1, uu = cc >> 1;
                if (tc3::EPI == 2 && (int)ub != grp) continue;  // the other group's accumulator
                tc::mbar_wait(b_tfull + 8 * ub, uu & 1);
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#ifdef BN_GRAM_PROBE_NOEPI  // timing probe (not product): no TMEM reads, no stores
                if (true) {
                    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
                    mbar_arrive(b_tempty + 8 * ub);
                    continue;
                }
#endif
                // x-wrapping chunks (not y-wrapping) hold their B rows group-major: column (gx, row, px)
                const bool gmaj = (x0 < 8 || x0 + 16 > L) && y0 + CH_ROWS * (ch + 1) <= L;
                for (int nyl = 0; nyl < CH_ROWS; ++nyl) {
                    const int ny = CH_ROWS * ch + nyl, oy = ny - dy;
                    uint32_t rc[32], rn[32];
                    const uint32_t tb = tmem + ((uint32_t)(32 * wq) << 16) + 256 * ub;
                    if (!gmaj) {
                        const uint32_t ta = tb + nyl * NBX;
                        tc::ld32(ta, rc);                       // <v_p, c_q>, q in x0-8 .. x0+23 of row ny
                        tc::ld32(ta + CH_ROWS * NBX, rn);       // <v_p, cn_q>
                    } else {
#pragma unroll
                        for (int gx = 0; gx < GRP; ++gx) {
                            const uint32_t ta = tb + (gx * CH_ROWS + nyl) * 8;
                            tc::ld8(ta, rc + 8 * gx);
                            tc::ld8(ta + CH_ROWS * NBX, rn + 8 * gx);
                        }
                    }
                    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                    if (oy < 0 || oy > R) continue;
                    int dc[2 * R + 1], dn[2 * R + 1];
#pragma unroll
                    for (int j = 0; j < NBX; ++j) scr[j] = fp ? __float2int_rz(__uint_as_float(rc[j])) : (int)rc[j];
#pragma unroll
                    for (int i = 0; i < 2 * R + 1; ++i) dc[i] = scr[dx + 8 - R + i];
#pragma unroll
                    for (int j = 0; j < NBX; ++j) scr[j] = fp ? __float2int_rz(__uint_as_float(rn[j])) : (int)rn[j];
#pragma unroll
                    for (int i = 0; i < 2 * R + 1; ++i) dn[i] = scr[dx + 8 - R + i];
                    // the row's 2R+1 records (+ zero pads) are whole 32-byte sectors of plane v:
                    // ru4(2R+1)/4 256-bit stores (ru4(R)/4 for the oy = 0 row, ox = 1..R)
                    int vx[NV], vy[NV];
#pragma unroll
                    for (int i = 0; i < NV; ++i) {
                        if (i < 2 * R + 1) {
                            const int nx = dx + 8 - R + i;
                            vx[i] = np + snorm[ny * NBX + nx] - 2 * dc[i];
                            vy[i] = np + snorm[(NBR + ny) * NBX + nx] - 2 * dn[i];
                        } else {
                            vx[i] = vy[i] = 0;
                        }
                    }
                    if (oy > 0) {
                        int2* o = out2 + hpad_index(-R, oy, R);
#pragma unroll
                        for (int q = 0; q < RW / 4; ++q) st_v8(o + 4 * q, vx + 4 * q, vy + 4 * q);
                    } else {
#pragma unroll
                        for (int q = 0; q < R0 / 4; ++q) st_v8(out2 + 4 * q, vx + R + 1 + 4 * q, vy + R + 1 + 4 * q);
                    }
                }
                asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
                mbar_arrive(b_tempty + 8 * ub);
            }
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
    }
    if (sched && threadIdx.x == 0) {  // the last CTA out resets the work counter for the next launch
        __threadfence();
        if (atomicAdd(sched + 1, 1u) == gridDim.x - 1) {
            sched[0] = 0;
            sched[1] = 0;
        }
    }
}

// ----------------------------------------------------------------------------- decisions
// Colour class s of pass t: one warp per active index m (SWAP: the lower index of a couple).
// dE_p = 2 * sum_{o in W} (acc[p+o] ? d1 : d0)[p][o]; accept iff dE < 0.
template <int R>
__device__ __forceinline__ i128 window_sum(const DTabs T, const uint8_t* __restrict__ acc, uint32_t L, uint32_t p) {
    constexpr int WN = (2 * R + 1) * (2 * R + 1) - 1;
    const int lane = threadIdx.x & 31;
    const uint32_t x = p % L, y = p / L;
    i128 s = 0;
    for (int w = lane; w < WN; w += 32) {
        const int ww = w >= R * (2 * R + 1) + R ? w + 1 : w;
        const int oy = ww / (2 * R + 1) - R, ox = ww % (2 * R + 1) - R;
        const uint32_t q = ((y + oy + L) & (L - 1)) * L + ((x + ox + L) & (L - 1));
        const size_t idx = (size_t)p * WN + w;
        const longlong2 t = T.d[idx];
        s += acc[q] ? get_term(t.y, T.x1, idx) : get_term(t.x, T.x0, idx);
    }
#pragma unroll
    for (int off = 16; off; off >>= 1) {
        const unsigned long long lo = __shfl_xor_sync(0xffffffffu, (unsigned long long)s, off);
        const long long hi = __shfl_xor_sync(0xffffffffu, (long long)(s >> 64), off);
        s += ((i128)hi << 64) | (u128)lo;
    }
    return s;
}

template <int R>
__global__ void k_decide(uint32_t s, uint32_t pass_t, uint64_t seed, uint32_t L, int mode, const DTabs T,
                         uint8_t* __restrict__ acc, i128* __restrict__ dEp, uint8_t* __restrict__ log) {
    const uint32_t M = (L / 8) * (L / 8);
    const uint32_t m = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (m >= M) return;
    const uint32_t p = class_pixel(L, seed, pass_t, s, m);
    if (mode == 0) {
        const i128 dE = 2 * window_sum<R>(T, acc, L, p);
        if ((threadIdx.x & 31) == 0) {
            const bool ok = dE < 0;
            acc[p] = ok;
            dEp[p] = ok ? dE : (i128)0;
            if (log) log[(size_t)s * M + m] = ok;
        }
    } else {
        const uint32_t mm = m ^ swap_kappa(seed, pass_t, s, M);
        if (mm < m) return;
        const uint32_t p2 = class_pixel(L, seed, pass_t, s, mm);
        const i128 dE = 2 * (window_sum<R>(T, acc, L, p) + window_sum<R>(T, acc, L, p2));
        if ((threadIdx.x & 31) == 0) {
            const bool ok = dE < 0;
            acc[p] = ok;
            acc[p2] = ok;
            dEp[p] = ok ? dE : (i128)0;
            dEp[p2] = 0;
            if (log) {
                log[(size_t)s * M + m] = ok;
                log[(size_t)s * M + mm] = ok;
            }
        }
    }
}

// Persistent decision kernel: all 64 colour classes of a pass in ONE cooperative launch.
// A "band" is the 8 lines (rows for even t, columns for odd t) holding active indices
// m = b*(L/8) + a of one b.  CTA g owns bands [g*G, (g+1)*G).  Class s of band b only depends
// on decisions of classes < s in bands b-1, b, b+1 (window radius R < 8), so CTA g waits until
// its neighbour CTAs have published progress >= s (no grid-wide barrier).  SWAP couples can
// straddle far bands: both owners evaluate the couple (identical, deterministic result) and
// each writes its own pixel's flag, after waiting on the bands around both members.
// The dE terms of the next candidate are loaded before the wait (they do not depend on it).
__device__ __forceinline__ int ld_acquire(const int* p) {
    int v;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release(int* p, int v) {
    asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

template <int R>
struct WinTerms {
    static constexpr int WN = (2 * R + 1) * (2 * R + 1) - 1;
    static constexpr int PER = (WN + 31) / 32;
    long long v0[PER], v1[PER];
    // from the shared-memory staging buffer: a row of WN {delta0, delta1} pairs
    __device__ __forceinline__ void load_smem(const long long* row) {
        const int lane = threadIdx.x & 31;
#pragma unroll
        for (int j = 0; j < PER; ++j) {
            const int w = lane + 32 * j;
            if (w < WN) {
                const longlong2 t = reinterpret_cast<const longlong2*>(row)[w];
                v0[j] = t.x;
                v1[j] = t.y;
            }
        }
    }
    // sum_w (acc[p + o_w] ? d1 : d0), reduced over the warp (every lane gets the total); exact in
    // int64 (R15: |term| < 2^55, |sum| < 2^63)
    __device__ __forceinline__ i128 sum(const uint8_t* acc, uint32_t L, uint32_t p, const DTabs T) const {
        const int lane = threadIdx.x & 31;
        const uint32_t x = p % L, y = p / L;
        uint8_t f[PER];
#pragma unroll
        for (int j = 0; j < PER; ++j) {
            const int w = lane + 32 * j;
            f[j] = 0;
            if (w < WN) {
                const int ww = w >= R * (2 * R + 1) + R ? w + 1 : w;
                const int oy = ww / (2 * R + 1) - R, ox = ww % (2 * R + 1) - R;
                const uint32_t q = ((y + oy + L) & (L - 1)) * L + ((x + ox + L) & (L - 1));
                f[j] = __ldcg(acc + q);
            }
        }
        long long s = 0;
#pragma unroll
        for (int j = 0; j < PER; ++j) {
            const int w = lane + 32 * j;
            if (w < WN) s += f[j] ? v1[j] : v0[j];
        }
#pragma unroll
        for (int off = 16; off; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
        return (i128)s;
    }
};

// Stage the dE-term rows (delta0, delta1) of the candidates of CTA `g` for class s into smem.
// Slot j holds candidate m = first + j (and, for SWAP, slot cpc + j its partner's rows); warp w
// copies slots w, w + nwarps, ... (row = WN {delta0, delta1} int64 pairs).
template <int R>
__device__ __forceinline__ void stage_class(uint32_t smem_base, const uint32_t* slot_pix, uint32_t nslot,
                                            const DTabs T) {
    constexpr int WN = WinTerms<R>::WN, NC = WN;  // 16-B chunks ({delta0, delta1} pairs) per table row
    const uint32_t warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5, lane = threadIdx.x & 31;
    for (uint32_t slot = warp; slot < nslot; slot += nwarps) {
        const size_t off = (size_t)slot_pix[slot] * WN;
        const uint32_t dst = smem_base + slot * 2 * WN * 8;
#pragma unroll
        for (uint32_t c = lane; c < (uint32_t)NC; c += 32) {
            cp_async16(dst + c * 16, T.d + off + c);
        }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
}

// Persistent decision kernel (REDRAW only; SWAP partners lie in far bands whose readers the
// progress protocol does not track): CTA g owns `cpc` consecutive active indices (a contiguous part
// of one band).  For class s it (1) moves the staged dE terms of its candidates from smem to
// registers, (2) immediately stages class s+1's terms with cp.async (they do not depend on any
// decision), (3) waits until the CTAs of the neighbouring bands have published progress >= s,
// (4) reads the neighbours' accept flags, reduces, decides, and publishes progress s+1.
template <int R, int mode>
__global__ void __launch_bounds__(512, 1) k_decide_pass(uint32_t pass_t, uint64_t seed, uint32_t L,
                                                        uint32_t cpc, const DTabs T, uint8_t* acc,
                                                        i128* __restrict__ dEp, uint8_t* __restrict__ log,
                                                        int* progress) {
    constexpr int WN = WinTerms<R>::WN;
    extern __shared__ __align__(16) uint8_t dsm[];
    __shared__ uint8_t sDelta[8 * 512];     // delta(t, r, b) & 7, r < 8, b < nb <= 512
    __shared__ uint32_t sKappa[64];
    __shared__ uint32_t sSlot[2][32];       // pixels of the staged slots, double indexed by class parity
    const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(dsm);
    const long long* srows = reinterpret_cast<const long long*>(dsm);
    const uint32_t nb = L / 8, M = nb * nb;
    const uint32_t g = blockIdx.x, ncta = gridDim.x, per_band = nb / cpc;
    const uint32_t first = g * cpc, nslot = mode ? 2 * cpc : cpc;
    const uint32_t warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    for (uint32_t j = threadIdx.x; j < 8 * nb; j += blockDim.x)
        sDelta[j] = (uint8_t)(philox_seeded(seed, j % nb, pass_t, j / nb, 2).x & 7);
    if (mode)
        for (uint32_t j = threadIdx.x; j < 64; j += blockDim.x) sKappa[j] = swap_kappa(seed, pass_t, j, M);
    __syncthreads();
    auto slot_pixels = [&](uint32_t s, uint32_t* out) {
        if (threadIdx.x < nslot) {
            const uint32_t j = threadIdx.x;
            const uint32_t m = j < cpc ? first + j : ((first + j - cpc) ^ sKappa[s]);
            out[j] = class_pixel_tab(sDelta, L, pass_t, s, m);
        }
    };
    slot_pixels(0, sSlot[0]);
    __syncthreads();
    stage_class<R>(sbase, sSlot[0], nslot, T);
    for (uint32_t s = 0; s < 64; ++s) {
        if (s + 1 < 64) slot_pixels(s + 1, sSlot[(s + 1) & 1]);
        asm volatile("cp.async.wait_group 0;" ::: "memory");
        __syncthreads();
        // warp j owns candidate first + j (the launch has exactly cpc warps)
        const uint32_t j = warp;
        const uint32_t kappa = mode ? sKappa[s] : 0;
        const uint32_t m = first + j, mm = m ^ kappa;
        const uint32_t p = sSlot[s & 1][j], p2 = mode ? sSlot[s & 1][cpc + j] : p;
        WinTerms<R> A, B;
        A.load_smem(srows + (size_t)j * 2 * WN);
        if (mode) B.load_smem(srows + (size_t)(cpc + j) * 2 * WN);
        __syncthreads();
        if (s + 1 < 64) stage_class<R>(sbase, sSlot[(s + 1) & 1], nslot, T);
        if (lane == 0 && s > 0) {
            const uint32_t bs[2] = {m / nb, mm / nb};
            for (int t = 0; t < (mode ? 2 : 1); ++t)
                for (int db = -1; db <= 1; ++db) {
                    const uint32_t bb = (bs[t] + nb + db) % nb;
                    for (uint32_t h = 0; h < per_band; ++h) {
                        const uint32_t owner = bb * per_band + h;
                        if (owner == g) continue;
                        while (ld_acquire(progress + owner) < (int)s) __nanosleep(20);
                    }
                }
        }
        __syncwarp();
        __threadfence();
        i128 sum = A.sum(acc, L, p, T);
        if (mode) sum += B.sum(acc, L, p2, T);
        const i128 dE = 2 * sum;
        if (lane == 0) {
            const bool ok = dE < 0;
            acc[p] = ok;
            dEp[p] = (ok && (!mode || m < mm)) ? dE : (i128)0;
            if (log) log[(size_t)s * M + m] = ok;
        }
        __threadfence();
        __syncthreads();
        if (threadIdx.x == 0 && ncta > 1) st_release(progress + g, (int)s + 1);
    }
}

// Cluster decision kernel (tiles with L*L/cpc <= 16 CTAs, i.e. L <= 128): the whole tile's
// accept flags live in every CTA's shared memory; after deciding class s each CTA pushes its
// new flags into every other CTA's copy through distributed shared memory (st.shared::cluster)
// and the cluster barrier (arrive.release / wait.acquire) orders them before class s+1.  No
// global-memory handshake is on the 64-class critical path.
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void st_cluster_u8(uint32_t local_addr, uint32_t cta, uint8_t v) {
    uint32_t remote;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(local_addr), "r"(cta));
    asm volatile("st.shared::cluster.u8 [%0], %1;" ::"r"(remote), "h"((unsigned short)v) : "memory");
}

// Per-lane window offsets (oy, ox) of the lane's terms w = lane + 32 j, computed once.
template <int R>
struct LaneOffsets {
    static constexpr int WN = WinTerms<R>::WN, PER = WinTerms<R>::PER;
    int oy[PER], ox[PER];
    int d[PER];  // oy * L + ox: the neighbour's pixel offset when the window does not wrap
    __device__ __forceinline__ void init(uint32_t L = 0) {
        const int lane = threadIdx.x & 31;
#pragma unroll
        for (int j = 0; j < PER; ++j) {
            const int w = lane + 32 * j;
            const int ww = w >= R * (2 * R + 1) + R ? w + 1 : w;
            oy[j] = w < WN ? ww / (2 * R + 1) - R : 0;
            ox[j] = w < WN ? ww % (2 * R + 1) - R : 0;
            d[j] = oy[j] * (int)L + ox[j];
        }
    }
};

// Cluster decision kernels (k_decide_cl3, k_decide_swap, k_decide_big): one 16-CTA cluster decides
// all 64 classes of a pass with no cluster barrier per class.  After deciding class s every warp
// pushes its pixel's accept flag (u32, 0 or 1) into every CTA's flag array with st.async, which also
// completes 4 bytes of transaction on that CTA's mailbox mbarrier for the class parity; a CTA starts
// class s+1 once its mailbox has received all M flags of class s.  A CTA can only send class s+1
// flags after receiving every flag of class s, i.e. after every warp of the cluster has finished
// reading the flags for class s, so a flag never changes under a reader.  The cluster-scope release
// of barrier.cluster.arrive (MEMBAR.ALL.GPU) is off the 64-class critical path.  (Round-1 variants
// with a cluster barrier per class or shared-memory-staged rows were measured slower and removed.)
template <int R>
struct WinTermsFlags32 : WinTerms<R> {
    // the candidate's delta0 / delta1 rows straight from global memory (read once: no L1 allocation)
    __device__ __forceinline__ void load_global(const DTabs T, uint32_t pix) {
        constexpr int WN = WinTerms<R>::WN, PER = WinTerms<R>::PER;
        const int lane = threadIdx.x & 31;
        const longlong2* r = T.d + (size_t)pix * WN;
#pragma unroll
        for (int j = 0; j < PER; ++j) {
            const int w = lane + 32 * j;
            if (w < WN)
                asm volatile("ld.global.nc.L1::no_allocate.v2.b64 {%0, %1}, [%2];"
                             : "=l"(this->v0[j]), "=l"(this->v1[j])
                             : "l"(r + w));
        }
    }
    // the same rows while other CTAs of the running kernel may still be writing other rows of the
    // table (k_pass_tail): L2-coherent loads, ordered after the producer's release by an acquire
    __device__ __forceinline__ void load_global_cg(const DTabs T, uint32_t pix) {
        constexpr int WN = WinTerms<R>::WN, PER = WinTerms<R>::PER;
        const int lane = threadIdx.x & 31;
        const longlong2* r = T.d + (size_t)pix * WN;
#pragma unroll
        for (int j = 0; j < PER; ++j) {
            const int w = lane + 32 * j;
            if (w < WN)
                asm volatile("ld.global.cg.v2.b64 {%0, %1}, [%2];" : "=l"(this->v0[j]), "=l"(this->v1[j]) : "l"(r + w)
                             : "memory");
        }
    }
    // exact int64 window sum (|term| < 2^55, <= 224 terms: |sum| < 2^63), warp-reduced in int64
    __device__ __forceinline__ i128 sum_flags(const uint32_t* sflags, uint32_t L, uint32_t p,
                                              const LaneOffsets<R>& off, const DTabs T) const {
        constexpr int WN = WinTerms<R>::WN, PER = WinTerms<R>::PER;
        const int lane = threadIdx.x & 31;
        const uint32_t x = p & (L - 1), y = p & ~(L - 1);
        long long acc = 0;
#pragma unroll
        for (int j = 0; j < PER; ++j) {
            const int w = lane + 32 * j;
            if (w < WN) {
                const uint32_t q = ((y + (uint32_t)off.oy[j] * L) & (L * L - 1)) + ((x + off.ox[j]) & (L - 1));
                acc += sflags[q] != 0 ? this->v1[j] : this->v0[j];
            }
        }
        return (i128)warp_sum_i64(acc);
    }
};

__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                 "l"(src), "r"(bytes), "r"(bar)
                 : "memory");
}
__device__ __forceinline__ void st_async_u32(uint32_t local_addr, uint32_t local_bar, uint32_t cta, uint32_t v) {
    uint32_t ra, rb;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(local_addr), "r"(cta));
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rb) : "r"(local_bar), "r"(cta));
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.u32 [%0], %1, [%2];" ::"r"(ra), "r"(v), "r"(rb)
                 : "memory");
}

__device__ __forceinline__ void red_async_or(uint32_t local_addr, uint32_t local_bar, uint32_t cta, uint32_t v) {
    uint32_t ra, rb;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(local_addr), "r"(cta));
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rb) : "r"(local_bar), "r"(cta));
    asm volatile("red.async.relaxed.cluster.shared::cluster.mbarrier::complete_tx::bytes.or.b32 [%0], %1, [%2];" ::"r"(ra),
                 "r"(v), "r"(rb)
                 : "memory");
}
template <int R>
struct WinTermsBits : WinTermsFlags32<R> {
    __device__ __forceinline__ long long sum_bits(const uint32_t* sbits, uint32_t L, uint32_t p,
                                                  const LaneOffsets<R>& off) const {
        constexpr int WN = WinTerms<R>::WN, PER = WinTerms<R>::PER;
        const int lane = threadIdx.x & 31;
        const uint32_t x = p & (L - 1), y = p & ~(L - 1);
        long long acc = 0;
        // the window does not wrap (warp-uniform): neighbour = p + oy L + ox, one add per term
        const bool inner = x >= (uint32_t)R && x + R < L && y >= (uint32_t)R * L && y + R * L < L * L;
        if (inner) {
#pragma unroll
            for (int j = 0; j < PER; ++j) {
                const int w = lane + 32 * j;
                if (w < WN) {
                    const uint32_t q = p + (uint32_t)off.d[j];
                    acc += (sbits[q >> 5] >> (q & 31)) & 1u ? this->v1[j] : this->v0[j];
                }
            }
        } else {
#pragma unroll
            for (int j = 0; j < PER; ++j) {
                const int w = lane + 32 * j;
                if (w < WN) {
                    const uint32_t q = ((y + (uint32_t)off.oy[j] * L) & (L * L - 1)) + ((x + off.ox[j]) & (L - 1));
                    acc += (sbits[q >> 5] >> (q & 31)) & 1u ? this->v1[j] : this->v0[j];
                }
            }
        }
        return warp_sum_i64(acc);
    }
};
// Cluster decision kernel v3: as v2 (st.async flag mailboxes, no cluster barrier) but every warp
// loads its candidate's dE-term rows for the next class straight into registers (issued one
// class ahead, so the L2 latency hides behind the current class) instead of staging them in
// shared memory: the shared-memory pipe, which bounds v2's window sums (57 KB of rows written and
// read back per class and SM), only serves the accept flags.
template <int R, int mode>
__global__ void __launch_bounds__(mode ? 256 : 512, 1) k_decide_cl3(uint32_t pass_t, uint64_t seed, uint32_t L, uint32_t cpc,
                                                       const DTabs T, uint8_t* __restrict__ acc,
                                                       i128* __restrict__ dEp, uint8_t* __restrict__ log) {
    constexpr uint32_t NSW = mode ? 2 : 1;  // candidates per warp (SWAP: the candidate and its partner)
    extern __shared__ __align__(16) uint8_t dsm[];
    __shared__ uint8_t sDelta[8 * 16];
    __shared__ uint32_t sKappa[64];
    __shared__ __align__(8) uint64_t sbar[2];  // mailboxes by class parity
    const uint32_t nb = L / 8, M = nb * nb, P = L * L;
    const uint32_t ncta = gridDim.x, first = blockIdx.x * cpc;
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    uint32_t* sflags = reinterpret_cast<uint32_t*>(dsm);  // [P]
    uint32_t* sSlot = sflags + P;                          // [64][cpc * NSW]
    const uint32_t sflags_addr = (uint32_t)__cvta_generic_to_shared(dsm);
    const uint32_t bar0 = (uint32_t)__cvta_generic_to_shared(&sbar[0]);
    auto mailbox = [&](uint32_t s) { return bar0 + 8 * (s & 1); };
    for (uint32_t j = threadIdx.x; j < P / 32; j += blockDim.x) sflags[j] = 0;  // accept bits
    for (uint32_t j = threadIdx.x; j < 8 * nb; j += blockDim.x)
        sDelta[j] = (uint8_t)(philox_seeded(seed, j % nb, pass_t, j / nb, 2).x & 7);
    if (mode)
        for (uint32_t j = threadIdx.x; j < 64; j += blockDim.x) sKappa[j] = swap_kappa(seed, pass_t, j, M);
    if (threadIdx.x == 0) {
        for (int i = 0; i < 2; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar0 + 8 * i) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const uint32_t per_class = cpc * NSW;
    for (uint32_t j = threadIdx.x; j < 64 * per_class; j += blockDim.x) {
        const uint32_t s = j / per_class, i = j - s * per_class;
        const uint32_t m = i < cpc ? first + i : ((first + i - cpc) ^ sKappa[s]);
        sSlot[j] = class_pixel_tab(sDelta, L, pass_t, s, m);
    }
    __syncthreads();
    WinTermsBits<R> A, B, An, Bn;
    A.load_global(T, sSlot[warp]);
    if (mode) B.load_global(T, sSlot[cpc + warp]);
    LaneOffsets<R> off;
    off.init(L);
    cluster_sync_all();  // every CTA's barriers and flags are initialised before any remote st.async
    for (uint32_t s = 0; s < 64; ++s) {
        if (s + 1 < 64) {  // next class's rows: in flight while this class waits and sums
            An.load_global(T, sSlot[(s + 1) * per_class + warp]);
            if (mode) Bn.load_global(T, sSlot[(s + 1) * per_class + cpc + warp]);
        }
        if (s > 0) tc::mbar_wait(mailbox(s - 1), ((s - 1) >> 1) & 1);  // all flags of class s-1
        if (threadIdx.x == 0)  // this CTA expects M flags of class s (the phase of class s-2 is complete)
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mailbox(s)), "r"(4 * M)
                         : "memory");
        const uint32_t m = first + warp, mm = m ^ (mode ? sKappa[s] : 0u);
        const uint32_t p = sSlot[s * per_class + warp], p2 = mode ? sSlot[s * per_class + cpc + warp] : p;
        BN_ASSERT(p < P && p2 < P);
        i128 sum = (i128)A.sum_bits(sflags, L, p, off);
        if (mode) sum += (i128)B.sum_bits(sflags, L, p2, off);
        const bool ok = 2 * sum < 0;
        if (lane < ncta) red_async_or(sflags_addr + 4 * (p >> 5), mailbox(s), lane, ok ? 1u << (p & 31) : 0u);
        if (lane == 0) {  // bookkeeping for commit/stats
            acc[p] = ok;
            dEp[p] = (ok && (!mode || m < mm)) ? 2 * sum : (i128)0;
            if (log) log[(size_t)s * M + m] = ok;
        }
        A = An;
        if (mode) B = Bn;
    }
    tc::mbar_wait(mailbox(63), (63 >> 1) & 1);  // every flag sent to this CTA has landed
    cluster_sync_all();
}

// SWAP cluster decision kernel: one warp per couple MEMBER (not per couple), so SWAP decisions
// run with the same 16 warps x 16 CTAs shape and register budget as REDRAW.  The couples
// {m, m ^ kappa} of class s are listed by their lower member (bit h = msb(kappa) of m clear), two
// consecutive slots per couple, so both members of a couple sit in the same CTA, in warps 2j and
// 2j+1: each warp sums its own member's window (acc-dependent terms, as in v3), the pair exchanges
// the two int128 sums through shared memory under a 64-thread named barrier, and both decide on
// the identical total.  Flags are broadcast exactly as in v3 (one st.async per member).
__device__ __forceinline__ uint32_t couple_member(uint32_t c, uint32_t kappa, uint32_t upper) {
    const uint32_t h = 31u - __clz(kappa);
    const uint32_t m = ((c >> h) << (h + 1)) | (c & ((1u << h) - 1u));
    return upper ? m ^ kappa : m;
}
#ifndef BN_SWAP_BITS
#define BN_SWAP_BITS 1  // SWAP decisions with the accept flags as bits (fewer shared-memory bank conflicts)
#endif
// Progress counters of the fused pass tail (k_pass_tail): lut[s] counts the finished dE-term units
// of class s, dec[s] the decided members of class s; reset by the kernel's last CTA.
struct TailCounters {
    unsigned int lut[64], dec[64];
    unsigned int lut_next, com_next, ticket, pad;
};
__device__ __forceinline__ void wait_count(const unsigned int* c, unsigned int target) {
    for (uint32_t n = 0;; ++n) {
        unsigned int v;
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(c) : "memory");
        if (v >= target) break;
        if (n > (1u << 28)) __trap();  // never hang the GPU on a protocol bug
        if (n > 8) __nanosleep(32);
    }
}
__device__ __forceinline__ void red_release_add(unsigned int* c, unsigned int v) {
    asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(c), "r"(v) : "memory");
}

// Body of k_decide_swap.  With `tc` (the fused pass tail) the CTA has one extra warp, the publisher:
// the deciding warps count their class-s members in shared memory (release, CTA scope) after
// writing acc / dEp, and the publisher, once all of the CTA's members of class s are counted, makes
// them visible at GPU scope (fence) and adds them to tc->dec[s] -- so no deciding warp ever waits on
// a GPU-scope fence (which would also drain its in-flight row prefetch).  With upc > 0 the rows of
// class s are only loaded once tc->lut[s] reaches upc.
template <int R>
__device__ __forceinline__ void decide_swap_body(uint8_t* dsm, uint32_t pass_t, uint64_t seed, uint32_t L, uint32_t cpc,
                                                 const DTabs T, uint8_t* __restrict__ acc, i128* __restrict__ dEp,
                                                 uint8_t* __restrict__ log, TailCounters* tc, uint32_t upc) {
    __shared__ uint8_t sDelta[8 * 16];
    __shared__ __align__(8) uint64_t sbar[2];
    __shared__ __align__(16) unsigned long long sPart[16][2];
    __shared__ unsigned int sDecCnt[64], sKap[64];
    const uint32_t nb = L / 8, M = nb * nb, P = L * L;
    const uint32_t ncta = cpc ? (M / cpc) : 0, first = (blockIdx.x % ncta) * cpc;  // first slot of this CTA
    const uint32_t cta = blockIdx.x % ncta;
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    uint32_t* sflags = reinterpret_cast<uint32_t*>(dsm);        // [P]
    uint32_t* sSlot = sflags + P;                                // [64][cpc] pixels
    uint16_t* sIdx = reinterpret_cast<uint16_t*>(sSlot + 64 * cpc);  // [64][cpc] active indices m
    const uint32_t sflags_addr = (uint32_t)__cvta_generic_to_shared(dsm);
    const uint32_t bar0 = (uint32_t)__cvta_generic_to_shared(&sbar[0]);
    auto mailbox = [&](uint32_t s) { return bar0 + 8 * (s & 1); };
    for (uint32_t j = threadIdx.x; j < (BN_SWAP_BITS ? P / 32 : P); j += blockDim.x) sflags[j] = 0;
    for (uint32_t j = threadIdx.x; j < 8 * nb; j += blockDim.x)
        sDelta[j] = (uint8_t)(philox_seeded(seed, j % nb, pass_t, j / nb, 2).x & 7);
    for (uint32_t j = threadIdx.x; j < 64; j += blockDim.x) {
        sDecCnt[j] = 0;
        sKap[j] = swap_kappa(seed, pass_t, j, M);  // one Philox per class, not per slot
    }
    if (threadIdx.x == 0) {
        for (int i = 0; i < 2; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar0 + 8 * i) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    for (uint32_t j = threadIdx.x; j < 64 * cpc; j += blockDim.x) {
        const uint32_t s = j / cpc, i = first + (j - s * cpc);
        const uint32_t m = couple_member(i >> 1, sKap[s], i & 1);
        sSlot[j] = class_pixel_tab(sDelta, L, pass_t, s, m);
        sIdx[j] = (uint16_t)m;
    }
    __syncthreads();
    if (tc && warp == cpc) {  // the publisher warp (fused pass tail)
        cluster_sync_all();
        if (lane == 0) {
            const uint32_t cnt_addr = (uint32_t)__cvta_generic_to_shared(sDecCnt);
            for (uint32_t s = 0; s < 64; ++s) {
                for (uint32_t n = 0;; ++n) {
                    unsigned int v;
                    asm volatile("ld.acquire.cta.shared::cta.u32 %0, [%1];" : "=r"(v) : "r"(cnt_addr + 4 * s) : "memory");
                    if (v >= cpc) break;
                    if (n > (1u << 28)) __trap();
                }
                red_release_add(tc->dec + s, cpc);  // fence.acq_rel.gpu + add: the members' writes first
            }
        }
        __syncwarp();
        cluster_sync_all();
        return;
    }
#if BN_SWAP_BITS
    WinTermsBits<R> A, An;
#else
    WinTermsFlags32<R> A, An;
#endif
    auto load_rows = [&](WinTermsFlags32<R>& X, uint32_t s) {
        if (tc && upc) {
            if (lane == 0) wait_count(tc->lut + s, upc);
            __syncwarp();
            X.load_global_cg(T, sSlot[s * cpc + warp]);
        } else {
            X.load_global(T, sSlot[s * cpc + warp]);
        }
    };
    load_rows(A, 0);
    LaneOffsets<R> off;
    off.init(L);
    cluster_sync_all();  // every CTA's barriers and flags are initialised before any remote st.async
    const uint32_t upper = (first + warp) & 1, pair_bar = 1 + (warp >> 1);
    for (uint32_t s = 0; s < 64; ++s) {
        if (s + 1 < 64) load_rows(An, s + 1);
        if (s > 0) tc::mbar_wait(mailbox(s - 1), ((s - 1) >> 1) & 1);  // all flags of class s-1
        if (threadIdx.x == 0)
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mailbox(s)), "r"(4 * M)
                         : "memory");
        const uint32_t p = sSlot[s * cpc + warp];
        BN_ASSERT(p < P);
#if BN_SWAP_BITS
        const i128 mine = (i128)A.sum_bits(sflags, L, p, off);
#else
        const i128 mine = A.sum_flags(sflags, L, p, off, T);
#endif
        if (lane == 0) {
            sPart[warp][0] = (unsigned long long)mine;
            sPart[warp][1] = (unsigned long long)((u128)mine >> 64);
        }
        asm volatile("bar.sync %0, 64;" ::"r"(pair_bar) : "memory");
        const uint32_t o = warp ^ 1;
        const i128 other = (i128)(((u128)sPart[o][1] << 64) | sPart[o][0]);
        const i128 sum = upper ? other + mine : mine + other;
        const bool ok = 2 * sum < 0;
#if BN_SWAP_BITS
        if (lane < ncta) red_async_or(sflags_addr + 4 * (p >> 5), mailbox(s), lane, ok ? 1u << (p & 31) : 0u);
#else
        if (lane < ncta) st_async_u32(sflags_addr + 4 * p, mailbox(s), lane, ok ? 1u : 0u);
#endif
        if (lane == 0) {
            acc[p] = ok;
            dEp[p] = (ok && !upper) ? 2 * sum : (i128)0;
            if (log) log[(size_t)s * M + sIdx[s * cpc + warp]] = ok;
            if (tc)  // counted for the publisher warp (release at CTA scope: acc / dEp written first)
                asm volatile("red.release.cta.shared::cta.add.u32 [%0], 1;" ::"r"(
                                 (uint32_t)__cvta_generic_to_shared(sDecCnt + s))
                             : "memory");
        }
        A = An;
    }
    (void)cta;
    tc::mbar_wait(mailbox(63), (63 >> 1) & 1);
    cluster_sync_all();
}
template <int R>
__global__ void __launch_bounds__(512, 1) k_decide_swap(uint32_t pass_t, uint64_t seed, uint32_t L, uint32_t cpc,
                                                        const DTabs T, uint8_t* __restrict__ acc,
                                                        i128* __restrict__ dEp, uint8_t* __restrict__ log) {
    extern __shared__ __align__(16) uint8_t dsm[];
    decide_swap_body<R>(dsm, pass_t, seed, L, cpc, T, acc, dEp, log, nullptr, 0);
}

// Cluster decisions for tiles with more candidates per class than one 16 x 16-warp cluster has
// warps (L = 256, 512): every warp owns `spw` consecutive slots of each class (REDRAW: candidates;
// SWAP: spw/2 whole couples, listed by their lower member, so a warp decides its couples alone),
// sums them one after another with the next slot's dE rows already in flight, and the pass's accept
// flags are BITS in shared memory (P/8 bytes: 8 KB for 256^2), broadcast with
// red.async.or.b32 ... mbarrier::complete_tx (4 bytes of transaction per candidate and CTA, sent
// whether 0 or 1).  Same mailbox protocol as k_decide_cl3.
// Body of k_decide_big.  With `tc` (the fused pass tail, SWAP) the CTA has one extra warp (warp
// nw), the publisher, exactly as in decide_swap_body: every lane that wrote a member's acc / dEp
// counts it in shared memory (release, CTA scope), and the publisher adds the CTA's cpc members of
// class s to tc->dec[s] at GPU scope once all are counted.
template <int R, int mode>
__device__ __forceinline__ void decide_big_body(uint8_t* dsm, uint32_t pass_t, uint64_t seed, uint32_t L, uint32_t spw,
                                                uint32_t nw, const DTabs T, uint8_t* __restrict__ acc,
                                                i128* __restrict__ dEp, uint8_t* __restrict__ log, TailCounters* tc) {
    __shared__ uint8_t sDelta[8 * 64];
    __shared__ __align__(8) uint64_t sbar[2];
    __shared__ unsigned int sDecCnt[64], sKap[64];
    const uint32_t nb = L / 8, M = nb * nb, P = L * L;
    const uint32_t ncta = M / (nw * spw), cpc = nw * spw;
    const uint32_t cta = blockIdx.x % ncta;
    const uint32_t first = cta * cpc;  // first slot of this CTA
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    uint32_t* sbits = reinterpret_cast<uint32_t*>(dsm);                 // [P / 32]
    uint32_t* sSlot = sbits + P / 32;                                   // [64][cpc] pixels
    uint16_t* sIdx = reinterpret_cast<uint16_t*>(sSlot + 64 * cpc);     // [64][cpc] active indices
    const uint32_t sbits_addr = (uint32_t)__cvta_generic_to_shared(dsm);
    const uint32_t bar0 = (uint32_t)__cvta_generic_to_shared(&sbar[0]);
    const uint32_t cnt_addr = (uint32_t)__cvta_generic_to_shared(sDecCnt);
    auto mailbox = [&](uint32_t s) { return bar0 + 8 * (s & 1); };
    for (uint32_t j = threadIdx.x; j < P / 32; j += blockDim.x) sbits[j] = 0;
    for (uint32_t j = threadIdx.x; j < 8 * nb; j += blockDim.x)
        sDelta[j] = (uint8_t)(philox_seeded(seed, j % nb, pass_t, j / nb, 2).x & 7);
    for (uint32_t j = threadIdx.x; j < 64; j += blockDim.x) {
        sDecCnt[j] = 0;
        if (mode) sKap[j] = swap_kappa(seed, pass_t, j, M);  // one Philox per class, not per slot
    }
    if (threadIdx.x == 0) {
        for (int i = 0; i < 2; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar0 + 8 * i) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    for (uint32_t j = threadIdx.x; j < 64 * cpc; j += blockDim.x) {
        const uint32_t s = j / cpc, i = first + (j - s * cpc);
        const uint32_t m = mode ? couple_member(i >> 1, sKap[s], i & 1) : i;
        sSlot[j] = class_pixel_tab(sDelta, L, pass_t, s, m);
        sIdx[j] = (uint16_t)m;
    }
    __syncthreads();
    if (tc && warp == nw) {  // the publisher warp (fused pass tail)
        cluster_sync_all();
        if (lane == 0) {
            for (uint32_t s = 0; s < 64; ++s) {
                for (uint32_t n = 0;; ++n) {
                    unsigned int v;
                    asm volatile("ld.acquire.cta.shared::cta.u32 %0, [%1];" : "=r"(v) : "r"(cnt_addr + 4 * s) : "memory");
                    if (v >= cpc) break;
                    if (n > (1u << 28)) __trap();
                }
                red_release_add(tc->dec + s, cpc);  // fence.acq_rel.gpu + add: the members' writes first
            }
        }
        __syncwarp();
        cluster_sync_all();
        return;
    }
    const uint32_t w0 = warp * spw;  // this warp's first slot within the CTA's slots of a class
    WinTermsBits<R> A, An;
    A.load_global(T, sSlot[w0]);
    LaneOffsets<R> off;
    off.init(L);
    cluster_sync_all();
    for (uint32_t s = 0; s < 64; ++s) {
        if (s > 0) tc::mbar_wait(mailbox(s - 1), ((s - 1) >> 1) & 1);  // all flags of class s-1
        if (threadIdx.x == 0)
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mailbox(s)), "r"(4 * M)
                         : "memory");
        long long prev = 0;  // SWAP: the lower member's window sum of the current couple
        for (uint32_t k = 0; k < spw; ++k) {
            // the next slot's rows (or the next class's first) are in flight while this one sums
            const bool more = k + 1 < spw || s + 1 < 64;
            if (more) An.load_global(T, sSlot[k + 1 < spw ? s * cpc + w0 + k + 1 : (s + 1) * cpc + w0]);
            const uint32_t slot = s * cpc + w0 + k, p = sSlot[slot];
            BN_ASSERT(p < P && slot < 64 * cpc);
            const long long mine = A.sum_bits(sbits, L, p, off);
            if (mode && !(k & 1)) {
                prev = mine;
            } else {
                const i128 sum = mode ? (i128)prev + (i128)mine : (i128)mine;
                const bool ok = 2 * sum < 0;
                const uint32_t np = mode ? 2 : 1;
                // flags of the decided member(s): lane l < np * ncta sends member l / ncta to CTA l % ncta
                if (lane < np * ncta) {
                    const uint32_t pk = sSlot[slot - (np - 1) + lane / ncta];
                    red_async_or(sbits_addr + 4 * (pk >> 5), mailbox(s), lane % ncta, ok ? 1u << (pk & 31) : 0u);
                }
                if (lane < np) {
                    const uint32_t sl = slot - (np - 1) + lane, pk = sSlot[sl];
                    acc[pk] = ok;
                    dEp[pk] = (ok && lane == 0) ? 2 * sum : (i128)0;
                    if (log) log[(size_t)s * M + sIdx[sl]] = ok;
                    if (tc)  // counted for the publisher warp (release at CTA scope: acc / dEp written first)
                        asm volatile("red.release.cta.shared::cta.add.u32 [%0], 1;" ::"r"(cnt_addr + 4 * s) : "memory");
                }
            }
            if (more) A = An;
        }
    }
    tc::mbar_wait(mailbox(63), (63 >> 1) & 1);
    cluster_sync_all();
}
template <int R, int mode>
__global__ void __launch_bounds__(512, 1) k_decide_big(uint32_t pass_t, uint64_t seed, uint32_t L, uint32_t spw,
                                                       const DTabs T, uint8_t* __restrict__ acc,
                                                       i128* __restrict__ dEp, uint8_t* __restrict__ log) {
    extern __shared__ __align__(16) uint8_t dsm[];
    decide_big_body<R, mode>(dsm, pass_t, seed, L, spw, blockDim.x >> 5, T, acc, dEp, log, nullptr);
}

// ------------------------------------------------------------------------------- pass sums
struct PassStatsDev {
    unsigned long long E_before[2];
    unsigned long long E_after[2];
    unsigned long long dE_sum[2];
    unsigned int accepted, pad;
};

// Single-CTA exact reductions: E_before = sum Epart, dE_sum = sum dEp, accepted = sum acc.
__global__ void __launch_bounds__(1024) k_pass_stats(const u128* __restrict__ Epart, uint32_t nEpart,
                                                     const i128* __restrict__ dEp, const uint8_t* __restrict__ acc,
                                                     uint32_t P, int swap_mode, PassStatsDev* __restrict__ out) {
    __shared__ unsigned long long s_e[1024][2], s_d[1024][2];
    __shared__ unsigned int s_a[1024];
    u128 e = 0;
    i128 d = 0;
    unsigned a = 0;
    for (uint32_t j = threadIdx.x; j < nEpart; j += blockDim.x) e += Epart[j];
    if (dEp)
        for (uint32_t j = threadIdx.x; j < P; j += blockDim.x) {
            d += dEp[j];
            a += acc[j];
        }
    s_e[threadIdx.x][0] = (unsigned long long)e;
    s_e[threadIdx.x][1] = (unsigned long long)(e >> 64);
    s_d[threadIdx.x][0] = (unsigned long long)(u128)d;
    s_d[threadIdx.x][1] = (unsigned long long)((u128)d >> 64);
    s_a[threadIdx.x] = a;
    __syncthreads();
    if (threadIdx.x == 0) {
        u128 E = 0, D = 0;
        unsigned A = 0;
        for (int j = 0; j < (int)blockDim.x; ++j) {
            E += ((u128)s_e[j][1] << 64) | s_e[j][0];
            D += ((u128)s_d[j][1] << 64) | s_d[j][0];
            A += s_a[j];
        }
        const u128 Ea = E + D;  // two's complement: E + dE_sum
        out->E_before[0] = (unsigned long long)E;
        out->E_before[1] = (unsigned long long)(E >> 64);
        out->E_after[0] = (unsigned long long)Ea;
        out->E_after[1] = (unsigned long long)(Ea >> 64);
        out->dE_sum[0] = (unsigned long long)D;
        out->dE_sum[1] = (unsigned long long)(D >> 64);
        out->accepted = swap_mode ? A / 2 : A;
    }
}

// Pass epilogue in one grid: commit accepted rows / shifts / norms, and the exact pass sums
// (E_before = sum Epart, dE_sum = sum dEp, accepted = sum acc) as per-block partials that the
// last block to finish (atomic ticket) reduces into `out`; the ticket is reset for the next use.
// Exact block-wide sums with 64-bit carries (warp shuffles, then warp 0 over the warps).
struct FinishPart {
    unsigned long long e[2], d[2];
    unsigned int a, pad[3];
};
__device__ __forceinline__ FinishPart block_sum_parts(u128 e, u128 d, unsigned a, FinishPart* s_w) {
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    e = warp_sum_u128(e);
    d = warp_sum_u128(d);
#pragma unroll
    for (int o = 16; o; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
    if (lane == 0) {
        s_w[warp].e[0] = (unsigned long long)e;
        s_w[warp].e[1] = (unsigned long long)(e >> 64);
        s_w[warp].d[0] = (unsigned long long)d;
        s_w[warp].d[1] = (unsigned long long)(d >> 64);
        s_w[warp].a = a;
    }
    __syncthreads();
    FinishPart r = {};
    if (warp == 0) {
        u128 E = 0, D = 0;
        unsigned A = 0;
        if (lane < nw) {
            E = ((u128)s_w[lane].e[1] << 64) | s_w[lane].e[0];
            D = ((u128)s_w[lane].d[1] << 64) | s_w[lane].d[0];
            A = s_w[lane].a;
        }
        E = warp_sum_u128(E);
        D = warp_sum_u128(D);
#pragma unroll
        for (int o = 16; o; o >>= 1) A += __shfl_xor_sync(0xffffffffu, A, o);
        r.e[0] = (unsigned long long)E;
        r.e[1] = (unsigned long long)(E >> 64);
        r.d[0] = (unsigned long long)D;
        r.d[1] = (unsigned long long)(D >> 64);
        r.a = A;
    }
    __syncthreads();  // s_w may be reused by the caller
    return r;
}
__global__ void __launch_bounds__(256) k_finish(const uint8_t* __restrict__ acc, uint32_t P, uint32_t rowB,
                                                uint32_t nl, const uint2* __restrict__ Un, uint2* __restrict__ U,
                                                const uint8_t* __restrict__ cn, uint8_t* __restrict__ c,
                                                const int* __restrict__ nn, int* __restrict__ nc,
                                                const u128* __restrict__ Epart, uint32_t nEpart,
                                                const i128* __restrict__ dEp, int swap_mode,
                                                FinishPart* __restrict__ parts, unsigned int* __restrict__ ticket,
                                                PassStatsDev* __restrict__ out, int clear_dEp,
                                                int check_prev, int* __restrict__ err) {
    const uint32_t nblk = gridDim.x, b = blockIdx.x;
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    const uint32_t p0 = (uint32_t)((uint64_t)P * b / nblk), p1 = (uint32_t)((uint64_t)P * (b + 1) / nblk);
    // commit: one warp per accepted pixel
    for (uint32_t p = p0 + warp; p < p1; p += nw) {
        if (!acc[p]) continue;
        const uint4* src = reinterpret_cast<const uint4*>(cn + (size_t)p * rowB);
        uint4* dst = reinterpret_cast<uint4*>(c + (size_t)p * rowB);
        for (uint32_t j = lane; j < rowB / 16; j += 32) dst[j] = src[j];
        if (lane == 0) U[p] = Un[p];
        if (lane < nl) nc[(size_t)p * nl + lane] = nn[(size_t)p * nl + lane];
    }
    // exact partial sums
    u128 e = 0;
    i128 d = 0;
    unsigned a = 0;
    const uint32_t e0 = (uint32_t)((uint64_t)nEpart * b / nblk), e1 = (uint32_t)((uint64_t)nEpart * (b + 1) / nblk);
    for (uint32_t j = e0 + threadIdx.x; j < e1; j += blockDim.x) e += Epart[j];
    i128* dEpw = const_cast<i128*>(dEp);  // the paper mode only rewrites its couples: clear after reading
    for (uint32_t j = p0 + threadIdx.x; j < p1; j += blockDim.x) {
        d += dEp[j];
        if (clear_dEp) dEpw[j] = 0;
        a += acc[j];
    }
    __shared__ FinishPart s_w[32];
    __shared__ bool last;
    FinishPart mine = block_sum_parts(e, (u128)d, a, s_w);  // (contains __syncthreads: commit reads done)
    // the next pass starts from all-zero accept flags (the per-class / flag-kernel decisions read
    // undecided neighbours' flags from acc)
    uint8_t* accw = const_cast<uint8_t*>(acc);
    for (uint32_t j = p0 + threadIdx.x; j < p1; j += blockDim.x) accw[j] = 0;
    if (threadIdx.x == 0) {
        parts[b] = mine;
        __threadfence();
        last = atomicAdd(ticket, 1u) == nblk - 1;
    }
    __syncthreads();
    if (!last) return;
    __threadfence();
    // the last block reduces all partials in parallel
    u128 E = 0, D = 0;
    unsigned A = 0;
    for (uint32_t j = threadIdx.x; j < nblk; j += blockDim.x) {
        const unsigned long long* q = reinterpret_cast<const unsigned long long*>(parts + j);
        E += ((u128)__ldcg(q + 1) << 64) | __ldcg(q + 0);
        D += ((u128)__ldcg(q + 3) << 64) | __ldcg(q + 2);
        A += (unsigned)__ldcg(q + 4);
    }
    const FinishPart tot = block_sum_parts(E, D, A, s_w);
    if (threadIdx.x == 0) {
        const u128 Et = ((u128)tot.e[1] << 64) | tot.e[0], Dt = ((u128)tot.d[1] << 64) | tot.d[0];
        const u128 Ea = Et + Dt;
        out->E_before[0] = tot.e[0];
        out->E_before[1] = tot.e[1];
        out->E_after[0] = (unsigned long long)Ea;
        out->E_after[1] = (unsigned long long)(Ea >> 64);
        out->dE_sum[0] = tot.d[0];
        out->dE_sum[1] = tot.d[1];
        out->accepted = swap_mode ? tot.a / 2 : tot.a;
        // exact energy chain: this pass's recomputed start energy equals the previous pass's
        // E_before + sum dE (greedy modes; the paper mode's snapshot swaps do not add up)
        if (check_prev && (__ldcg(&out[-1].E_after[0]) != tot.e[0] || __ldcg(&out[-1].E_after[1]) != tot.e[1]))
            atomicOr(err, 4);
        *ticket = 0;
    }
}

// ------------------------------------------------------ paper-verbatim parallel swaps (f1)
// PAPER.md §3.4 l.291-307: the couples of pass t are consecutive entries of a precomputed
// permutation of the pixel indices, XOR-scrambled with a per-pass key (l.303-306):
//   key(t) = Philox(seed; t, 0, 0, 5)[0] & (P - 1),  couple c = (perm[2c] ^ key, perm[2c+1] ^ key).
// Every couple is evaluated against the pass-start tile (l.294-295, snapshot reading R26) and
// every couple with dE < 0 is swapped; the couples are pixel-disjoint (l.293-294), so the commit
// is race-free.  The window distances of the snapshot come from the same Gram as the greedy
// path: with cn_p = c_partner(p), delta0[p][o] = sum_l q(o, D(cn_p, c_p+o)) - q(o, D(c_p, c_p+o))
// is exactly p's share of the couple's dE.
__device__ __forceinline__ uint32_t paper_key(uint64_t seed, uint32_t t, uint32_t P) {
    return philox_seeded(seed, t, 0, 0, 5).x & (P - 1u);
}
// Partner of pixel p in pass t's couples (p itself if p is in none): p sits at position
// j = invperm[p ^ key] of the scrambled sequence, and couples are consecutive positions.
__device__ __forceinline__ uint32_t paper_partner(const uint32_t* __restrict__ perm, const uint32_t* __restrict__ invperm,
                                                  uint32_t key, uint32_t budget, uint32_t p) {
    const uint32_t j = __ldg(invperm + (p ^ key));
    return j < budget ? __ldg(perm + (j ^ 1u)) ^ key : p;
}
// cn_p = c_part(p), Un_p = U_part(p), nn_p = nc_part(p); pixels outside every couple take their own
// rows (their dE terms are never read, but their distances must stay in the LUT range).
// One warp per pixel, 16-byte copies.
__global__ void k_paper_gather(const uint32_t* __restrict__ part, const uint2* __restrict__ U, uint2* __restrict__ Un,
                               const uint8_t* __restrict__ c, uint8_t* __restrict__ cn, const int* __restrict__ nc,
                               int* __restrict__ nn, uint32_t P, uint32_t rowB, uint32_t nl,
                               const uint32_t* __restrict__ perm = nullptr, const uint32_t* __restrict__ invperm = nullptr,
                               uint64_t seed = 0, uint32_t pass_t = 0, uint32_t budget = 0) {
    const uint32_t p = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
    if (p >= P) return;
    uint32_t q;
    if (part) {
        const uint32_t q0 = __ldg(part + p);
        q = q0 == 0xFFFFFFFFu ? p : q0;
    } else {  // paper mode: partner from the inverse permutation
        q = 0;
        if (lane == 0) q = paper_partner(perm, invperm, paper_key(seed, pass_t, P), budget, p);
        q = __shfl_sync(0xffffffffu, q, 0);
    }
    const uint4* src = reinterpret_cast<const uint4*>(c + (size_t)q * rowB);
    uint4* dst = reinterpret_cast<uint4*>(cn + (size_t)p * rowB);
    for (uint32_t j = lane; j < rowB / 16; j += 32) dst[j] = __ldg(src + j);
    if (lane == 0) Un[p] = U[q];
    if (lane < nl) nn[(size_t)p * nl + lane] = nc[(size_t)q * nl + lane];
}
// Snapshot window sum of p's delta0 terms, skipping the partner `skip` (its distance to p does
// not change under the swap).  Exact int128, warp-wide.
template <int R>
__device__ __forceinline__ i128 window_sum_snapshot(const DTabs T, uint32_t L, uint32_t p, uint32_t skip) {
    constexpr int WN = (2 * R + 1) * (2 * R + 1) - 1;
    const int lane = threadIdx.x & 31;
    const uint32_t x = p % L, y = p / L;
    long long s = 0;  // exact: every term < 2^55, every window sum < 2^63 (R15)
    for (int w = lane; w < WN; w += 32) {
        const int ww = w >= R * (2 * R + 1) + R ? w + 1 : w;
        const int oy = ww / (2 * R + 1) - R, ox = ww % (2 * R + 1) - R;
        const uint32_t q = ((y + oy + L) & (L - 1)) * L + ((x + ox + L) & (L - 1));
        if (q == skip) continue;
        s += __ldg(reinterpret_cast<const long long*>(T.d) + 2 * ((size_t)p * WN + w));  // delta0
    }
    return (i128)warp_sum_i64(s);
}
// One warp per couple: dE = 2 (sum_o' delta0[p][o] + sum_o' delta0[q][o]); accept iff dE < 0.
// acc marks both members (k_finish commits their gathered rows), dEp holds the couple's dE once.
// log[c] = accept flag of couple c.
template <int R>
__global__ void k_paper_decide(const uint32_t* __restrict__ perm, uint64_t seed, uint32_t pass_t, uint32_t L,
                               uint32_t ncp, const DTabs T, uint8_t* __restrict__ acc, i128* __restrict__ dEp,
                               uint8_t* __restrict__ log) {
    const uint32_t c = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (c >= ncp) return;
    const uint32_t P = L * L, key = paper_key(seed, pass_t, P);
    const uint32_t p = __ldg(perm + 2 * c) ^ key, q = __ldg(perm + 2 * c + 1) ^ key;
    const i128 dE = 2 * (window_sum_snapshot<R>(T, L, p, q) + window_sum_snapshot<R>(T, L, q, p));
    if ((threadIdx.x & 31) == 0) {
        const bool ok = dE < 0;
        acc[p] = ok;
        acc[q] = ok;
        dEp[p] = ok ? dE : (i128)0;
        dEp[q] = 0;
        if (log) log[c] = ok;
    }
}

// --------------------------------------------------- evaluation criterion
// PAPER.md §3.3 l.270-284 / teaser (c): RMSE of the test-integrand tiles after Gaussian
// denoising, for a range of kernel widths, and the error power spectrum.  Computed through the
// 2D DFT of every integrand's error image e_i(p) = c_i(p)/N - I_ref,i (fp64): the toroidal
// convolution is a product in frequency space, so by Parseval
//   rmse_i(sigma)^2 = 1/P^2 sum_f |E_i(f)|^2 K_sigma(f)^2,   K_sigma(kx,ky) = h(kx) h(ky)
// (h = DFT of the periodised, normalised 1D Gaussian; real and even), and the spectrum is
// |E_i(f)|^2 with the DC bin (the mean) removed.  Row DFT -> column DFT -> per-(integrand, kx)
// partial sums, reduced in a fixed order (deterministic).
constexpr int EV_II = 32;  // integrands per CTA
// X1[ii][kx][y] = sum_x e_ii(x, y) w^(kx x), w = exp(-2 pi i / L); one CTA per (row y, 32 integrands).
__global__ void __launch_bounds__(256) k_ev_dft_rows(const uint8_t* __restrict__ c, uint32_t L, uint32_t rowB,
                                                     uint32_t loff, double invN, const double* __restrict__ iref,
                                                     uint32_t i0, uint32_t ni, const double2* __restrict__ tw,
                                                     double2* __restrict__ X1, const double* __restrict__ img) {
    extern __shared__ double ev_smem[];
    double* E = ev_smem;                                         // [L][EV_II]
    double2* w = reinterpret_cast<double2*>(E + (size_t)L * EV_II);  // [L]
    const uint32_t y = blockIdx.x, ic = blockIdx.y * EV_II;      // chunk-local integrand base
    for (uint32_t j = threadIdx.x; j < L; j += blockDim.x) w[j] = tw[j];
    for (uint32_t j = threadIdx.x; j < L * EV_II; j += blockDim.x) {
        const uint32_t x = j / EV_II, ii = j % EV_II, i = ic + ii;
        // error image: from the counts (c / N - I_ref) or given (img [ni][P], the smooth family)
        E[j] = i >= ni ? 0.0
               : img  ? img[(size_t)(i0 + i) * L * L + y * L + x]
                      : (double)c[(size_t)(y * L + x) * rowB + loff + i0 + i] * invN - iref[i0 + i];
    }
    __syncthreads();
    for (uint32_t o = threadIdx.x; o < L * EV_II; o += blockDim.x) {
        const uint32_t kx = o / EV_II, ii = o % EV_II, i = ic + ii;
        double re = 0.0, im = 0.0;
        for (uint32_t x = 0; x < L; ++x) {
            const double2 t = w[(kx * x) & (L - 1)];
            const double e = E[x * EV_II + ii];
            re = fma(e, t.x, re);
            im = fma(e, t.y, im);
        }
        if (i < ni) X1[((size_t)i * L + kx) * L + y] = make_double2(re, im);
    }
}
// Column DFT of X1 for one kx and 32 integrands, power |E(kx, ky)|^2, then
//   rm[i][kx][s] = sum_ky |E|^2 K_s(kx, ky)^2       (partial Parseval sums)
//   sp[cta][ky][kx] = sum_{ii in CTA} |E|^2          (DC excluded; partial spectrum)
__global__ void __launch_bounds__(256) k_ev_dft_cols(const double2* __restrict__ X1, uint32_t L, uint32_t i0,
                                                     uint32_t ni, const double2* __restrict__ tw,
                                                     const double* __restrict__ h /* [ns][L] */, uint32_t ns,
                                                     double* __restrict__ rm, double* __restrict__ sp) {
    extern __shared__ double ev_smem[];
    double2* X = reinterpret_cast<double2*>(ev_smem);            // [L][EV_II]
    double2* w = X + (size_t)L * EV_II;                           // [L]
    double* pw = reinterpret_cast<double*>(w + L);                // [L][EV_II]
    const uint32_t kx = blockIdx.x, ic = blockIdx.y * EV_II;
    for (uint32_t j = threadIdx.x; j < L; j += blockDim.x) w[j] = tw[j];
    for (uint32_t j = threadIdx.x; j < L * EV_II; j += blockDim.x) {
        const uint32_t ii = j / L, y = j % L, i = ic + ii;
        X[y * EV_II + ii] = i < ni ? X1[((size_t)i * L + kx) * L + y] : make_double2(0.0, 0.0);
    }
    __syncthreads();
    for (uint32_t o = threadIdx.x; o < L * EV_II; o += blockDim.x) {
        const uint32_t ky = o / EV_II, ii = o % EV_II;
        double re = 0.0, im = 0.0;
        for (uint32_t y = 0; y < L; ++y) {
            const double2 t = w[(ky * y) & (L - 1)], v = X[y * EV_II + ii];
            re = fma(v.x, t.x, re);
            re = fma(-v.y, t.y, re);
            im = fma(v.x, t.y, im);
            im = fma(v.y, t.x, im);
        }
        pw[ky * EV_II + ii] = re * re + im * im;
    }
    __syncthreads();
    // Parseval partials: one thread per (integrand, sigma), fixed ky order
    for (uint32_t o = threadIdx.x; o < EV_II * ns; o += blockDim.x) {
        const uint32_t ii = o / ns, sg = o % ns, i = ic + ii;
        if (i >= ni) continue;
        const double hx = h[(size_t)sg * L + kx];
        double acc = 0.0;
        for (uint32_t ky = 0; ky < L; ++ky) {
            const double k2 = hx * h[(size_t)sg * L + ky];
            acc = fma(pw[ky * EV_II + ii], k2 * k2, acc);
        }
        rm[((size_t)(i0 + i) * L + kx) * ns + sg] = acc;
    }
    // spectrum partial over this CTA's integrands, fixed ii order
    for (uint32_t ky = threadIdx.x; ky < L; ky += blockDim.x) {
        double acc = 0.0;
        if (kx != 0 || ky != 0)
            for (uint32_t ii = 0; ii < EV_II; ++ii) acc += pw[ky * EV_II + ii];
        sp[((size_t)((i0 + ic) / EV_II) * L + ky) * L + kx] = acc;
    }
}
// rmse[s] = 1/Ts sum_i sqrt(sum_kx rm[i][kx][s]) / P  -- one CTA per sigma, exact fixed order per
// integrand, then a fixed-order block sum.
__global__ void __launch_bounds__(256) k_ev_rmse(const double* __restrict__ rm, uint32_t L, uint32_t Ts, uint32_t ns,
                                                 double* __restrict__ out) {
    __shared__ double part[256];
    const uint32_t sg = blockIdx.x;
    double acc = 0.0;
    for (uint32_t i = threadIdx.x; i < Ts; i += blockDim.x) {
        double s = 0.0;
        for (uint32_t kx = 0; kx < L; ++kx) s += rm[((size_t)i * L + kx) * ns + sg];
        acc += sqrt(s) / ((double)L * L);
    }
    part[threadIdx.x] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int j = 0; j < (int)blockDim.x; ++j) t += part[j];
        out[sg] = t / Ts;
    }
}
// spectrum[f] = 1/Ts sum_chunks sp[chunk][f]; profile[j] = mean of spectrum over floor(|f|) = j + 1.
__global__ void __launch_bounds__(256) k_ev_spectrum(const double* __restrict__ sp, uint32_t L, uint32_t nchunk,
                                                     uint32_t Ts, double* __restrict__ S, double* __restrict__ prof) {
    const uint32_t P = L * L;
    for (uint32_t f = threadIdx.x; f < P; f += blockDim.x) {
        double acc = 0.0;
        for (uint32_t k = 0; k < nchunk; ++k) acc += sp[(size_t)k * P + f];
        S[f] = acc / Ts;
    }
    __syncthreads();
    for (uint32_t j = threadIdx.x; j < L / 2; j += blockDim.x) {
        double sum = 0.0;
        uint32_t n = 0;
        for (uint32_t f = 0; f < P; ++f) {
            const int kx = (int)(f % L), ky = (int)(f / L);
            const int fx = kx <= (int)L / 2 ? kx : kx - (int)L, fy = ky <= (int)L / 2 ? ky : ky - (int)L;
            if ((uint32_t)floor(sqrt((double)(fx * fx + fy * fy))) == j + 1) {
                sum += S[f];
                ++n;
            }
        }
        prof[j] = n ? sum / n : 0.0;
    }
}

// SWAP pass epilogue fused with the next pass's gather: one warp per pixel p
//   commit:  acc[p] -> c_p <- cn_p, U_p <- Un_p, nc_p <- nn_p                    (this pass)
//   gather:  cn2_p <- row of src = part_next[p] in its post-commit state          (next pass)
//            = acc[src] ? cn_src : c_src  (c_src is only written here when acc[src], so every read
//            sees either an untouched c row or the candidate row: no ordering between warps needed)
// plus the exact pass sums of k_finish (per-block partials, last-block reduction), which also
// clears the accept flags once every block has read them.
#ifndef BN_FG_THREADS
#define BN_FG_THREADS 1024  // k_finish_gather block size
#endif
#ifndef BN_FG_MINB
#define BN_FG_MINB 1  // resident blocks per SM requested from ptxas
#endif
#ifndef BN_FG_BPS
#define BN_FG_BPS 1  // k_finish_gather blocks per SM in the grid (one wave: C3 commit 0.0395 -> 0.036 ms vs 2)
#endif
__global__ void __launch_bounds__(BN_FG_THREADS, BN_FG_MINB) k_finish_gather(uint8_t* __restrict__ acc, uint32_t P, uint32_t rowB,
                                                       uint32_t nl, const uint2* __restrict__ Un, uint2* __restrict__ U,
                                                       const uint8_t* __restrict__ cn, uint8_t* __restrict__ c,
                                                       const int* __restrict__ nn, int* __restrict__ nc,
                                                       const u128* __restrict__ Epart, uint32_t nEpart,
                                                       const i128* __restrict__ dEp,
                                                       FinishPart* __restrict__ parts, unsigned int* __restrict__ ticket,
                                                       PassStatsDev* __restrict__ out,
                                                       const uint32_t* __restrict__ part_next, uint2* __restrict__ Un2,
                                                       uint8_t* __restrict__ cn2, int* __restrict__ nn2, uint32_t L,
                                                       uint64_t seed, uint32_t pass_next,
                                                       const uint32_t* __restrict__ perm,
                                                       const uint32_t* __restrict__ invperm, uint32_t budget,
                                                       int check_prev, int* __restrict__ err) {
    const uint32_t nblk = gridDim.x, b = blockIdx.x;
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    const uint32_t n16 = rowB / 16;
    const uint32_t p0 = (uint32_t)((uint64_t)P * b / nblk), p1 = (uint32_t)((uint64_t)P * (b + 1) / nblk);
    for (uint32_t p = p0 + warp; p < p1; p += nw) {
        if (acc[p]) {
            const uint4* src = reinterpret_cast<const uint4*>(cn + (size_t)p * rowB);
            uint4* dst = reinterpret_cast<uint4*>(c + (size_t)p * rowB);
            for (uint32_t j = lane; j < n16; j += 32) dst[j] = src[j];
            if (lane == 0) U[p] = Un[p];
            if (lane < nl) nc[(size_t)p * nl + lane] = nn[(size_t)p * nl + lane];
        }
        uint32_t q = 0;
        if (lane == 0)
            q = part_next ? part_next[p]
                : perm    ? paper_partner(perm, invperm, paper_key(seed, pass_next, P), budget, p)
                          : swap_partner(L, seed, pass_next, p);
        q = __shfl_sync(0xffffffffu, q, 0);
        BN_ASSERT(q < P);
        const bool a = acc[q] != 0;
        const uint4* src = reinterpret_cast<const uint4*>((a ? cn : c) + (size_t)q * rowB);
        uint4* dst = reinterpret_cast<uint4*>(cn2 + (size_t)p * rowB);
        for (uint32_t j = lane; j < n16; j += 32) dst[j] = src[j];
        if (lane == 0) Un2[p] = a ? Un[q] : U[q];
        if (lane < nl) nn2[(size_t)p * nl + lane] = a ? nn[(size_t)q * nl + lane] : nc[(size_t)q * nl + lane];
    }
    // exact partial sums (this block's pixels, its share of Epart)
    u128 e = 0;
    i128 d = 0;
    unsigned na = 0;
    const uint32_t e0 = (uint32_t)((uint64_t)nEpart * b / nblk), e1 = (uint32_t)((uint64_t)nEpart * (b + 1) / nblk);
    for (uint32_t j = e0 + threadIdx.x; j < e1; j += blockDim.x) e += Epart[j];
    i128* dEpw = const_cast<i128*>(dEp);  // the paper mode only rewrites its couples: clear after reading
    for (uint32_t j = p0 + threadIdx.x; j < p1; j += blockDim.x) {
        d += dEp[j];
        if (perm) dEpw[j] = 0;
        na += acc[j];
    }
    __shared__ FinishPart s_w[32];
    __shared__ bool last;
    FinishPart mine = block_sum_parts(e, (u128)d, na, s_w);
    if (threadIdx.x == 0) {
        parts[b] = mine;
        __threadfence();
        last = atomicAdd(ticket, 1u) == nblk - 1;
    }
    __syncthreads();
    if (!last) return;
    __threadfence();
    u128 E = 0, D = 0;
    unsigned A = 0;
    for (uint32_t j = threadIdx.x; j < nblk; j += blockDim.x) {
        const unsigned long long* qq = reinterpret_cast<const unsigned long long*>(parts + j);
        E += ((u128)__ldcg(qq + 1) << 64) | __ldcg(qq + 0);
        D += ((u128)__ldcg(qq + 3) << 64) | __ldcg(qq + 2);
        A += (unsigned)__ldcg(qq + 4);
    }
    const FinishPart tot = block_sum_parts(E, D, A, s_w);
    // every block has read its accept flags (and every gather its sources'): clear them for the
    // next pass's decisions (uint4 stores; P is a multiple of 256)
    for (uint32_t j = threadIdx.x; j < P / 16; j += blockDim.x) reinterpret_cast<uint4*>(acc)[j] = make_uint4(0, 0, 0, 0);
    if (threadIdx.x == 0) {
        const u128 Et = ((u128)tot.e[1] << 64) | tot.e[0], Dt = ((u128)tot.d[1] << 64) | tot.d[0];
        const u128 Ea = Et + Dt;
        out->E_before[0] = tot.e[0];
        out->E_before[1] = tot.e[1];
        out->E_after[0] = (unsigned long long)Ea;
        out->E_after[1] = (unsigned long long)(Ea >> 64);
        out->dE_sum[0] = tot.d[0];
        out->dE_sum[1] = tot.d[1];
        out->accepted = tot.a / 2;
        if (check_prev && (__ldcg(&out[-1].E_after[0]) != tot.e[0] || __ldcg(&out[-1].E_after[1]) != tot.e[1]))
            atomicOr(err, 4);
        *ticket = 0;
    }
}

// ------------------------------------------------------------ fused pass tail (SWAP, 64 <= L <= 512)
// One cooperative launch of clusters of `ncta` CTAs replaces k_decide_swap + k_finish_gather
// (DESIGN.md §5.8).  Cluster 0 decides the 64 colour classes exactly as k_decide_swap and publishes
// every decided member in tc->dec[s]; the other clusters commit in class order behind it: once all
// M members of class s are decided, each member q's final row (acc ? cn_q : c_q) is committed and
// gathered into the next pass's candidate buffer at its next-pass partner, and the pass's exact
// sums are accumulated (the last helper reduces them).  Co-residency of the decision cluster and
// the helpers (which wait on it) is guaranteed by the cooperative launch.  Bit-identical to the
// separate kernels: the same decisions, the same copies, the same exact sums.
template <int R, bool BIG>
__global__ void __launch_bounds__(544, 1) k_pass_tail(uint32_t pass_t, uint64_t seed, uint32_t L, uint32_t cpc,
                                                      longlong2* __restrict__ dterms, uint8_t* __restrict__ acc,
                                                      i128* __restrict__ dEp, uint8_t* __restrict__ log,
                                                      const u128* __restrict__ Epart, uint32_t nEpart, uint32_t nl,
                                                      int* __restrict__ err,
                                                      uint32_t rowB, const uint2* __restrict__ Un, uint2* __restrict__ U,
                                                      const uint8_t* __restrict__ cn, uint8_t* __restrict__ c,
                                                      const int* __restrict__ nn, int* __restrict__ nc,
                                                      uint2* __restrict__ Un2, uint8_t* __restrict__ cn2,
                                                      int* __restrict__ nn2, int gather_next,
                                                      FinishPart* __restrict__ parts, PassStatsDev* __restrict__ out,
                                                      int check_prev, TailCounters* __restrict__ tc) {
    extern __shared__ __align__(16) uint8_t dsm[];
    constexpr int WN = (2 * R + 1) * (2 * R + 1) - 1;
    const uint32_t nb = L / 8, M = nb * nb, P = L * L;
    const uint32_t ncta = M / cpc;
    const DTabs T = {dterms, nullptr, nullptr};
    if (blockIdx.x < ncta) {  // cluster 0: the decisions
        if (BIG)  // L = 256, 512: cpc / 16 slots per warp (k_decide_big)
            decide_big_body<R, 1>(dsm, pass_t, seed, L, cpc / 16, 16, T, acc, dEp, log, tc);
        else
            decide_swap_body<R>(dsm, pass_t, seed, L, cpc, T, acc, dEp, log, tc, 0);
        return;
    }
    // ------------------------------------------------------------------------ helpers
    __shared__ uint8_t sD[8 * 64];  // nb <= 64
    __shared__ uint32_t sUnit;
    __shared__ FinishPart s_w[32];
    __shared__ bool last;
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t nh = gridDim.x - ncta, hb = blockIdx.x - ncta;
    for (uint32_t j = threadIdx.x; j < 8 * nb; j += blockDim.x)
        sD[j] = (uint8_t)(philox_seeded(seed, j % nb, pass_t, j / nb, 2).x & 7);
    __syncthreads();
    auto cls = [&](uint32_t q) -> uint32_t {  // colour class of pixel q in pass t
        const uint32_t x = q & (L - 1), y = q / L;
        const uint32_t along = (pass_t & 1) ? y : x, across = (pass_t & 1) ? x : y;
        const uint32_t r = across & 7;
        return 8 * r + ((along - sD[r * nb + (across >> 3)]) & 7);
    };
    // pass-start energy: this helper's share of the k_lut block partials
    u128 e = 0;
    const uint32_t e0 = (uint32_t)((uint64_t)nEpart * hb / nh), e1 = (uint32_t)((uint64_t)nEpart * (hb + 1) / nh);
    for (uint32_t j = e0 + threadIdx.x; j < e1; j += blockDim.x) e += Epart[j];
    // commit + next-pass gather in class order (unit = hw members, one per warp), exact sums
    const uint32_t hw = (blockDim.x >> 5) < 16 ? (blockDim.x >> 5) : 16;
    const uint32_t cpu_ = (M + hw - 1) / hw, ncunits = 64 * cpu_;
    i128 dsum = 0;
    unsigned na = 0;
    const uint32_t n16 = rowB / 16;
    for (;;) {
        if (threadIdx.x == 0) {
            sUnit = atomicAdd(&tc->com_next, 1u);
            if (sUnit < ncunits) wait_count(tc->dec + sUnit / cpu_, M);
        }
        __syncthreads();
        const uint32_t u = sUnit;
        __syncthreads();
        if (u >= ncunits) break;
        const uint32_t s = u / cpu_, m = (u - s * cpu_) * hw + warp;
        if (warp >= hw || m >= M) continue;
        const uint32_t q = class_pixel_tab(sD, L, pass_t, s, m);
        BN_ASSERT(q < P && s < 64);
        const bool a = __ldcg(acc + q) != 0;
        const uint4* src = reinterpret_cast<const uint4*>((a ? cn : c) + (size_t)q * rowB);
        uint32_t p2 = 0;
        if (gather_next) {
            if (lane == 0) p2 = swap_partner(L, seed, pass_t + 1, q);
            p2 = __shfl_sync(0xffffffffu, p2, 0);
            BN_ASSERT(p2 < P);
        }
        uint4* dst_c = reinterpret_cast<uint4*>(c + (size_t)q * rowB);
        uint4* dst_n = reinterpret_cast<uint4*>(cn2 + (size_t)p2 * rowB);
        for (uint32_t j = lane; j < n16; j += 32) {
            const uint4 v = src[j];
            if (a) dst_c[j] = v;
            if (gather_next) dst_n[j] = v;
        }
        if (lane == 0) {
            const uint2 uq = a ? Un[q] : U[q];
            if (a) U[q] = uq;
            if (gather_next) Un2[p2] = uq;
            const unsigned long long lo = __ldcg(reinterpret_cast<const unsigned long long*>(dEp + q));
            const unsigned long long hi = __ldcg(reinterpret_cast<const unsigned long long*>(dEp + q) + 1);
            dsum += (i128)(((u128)hi << 64) | lo);
            na += a;
            acc[q] = 0;  // the next pass starts from all-zero accept flags
        }
        if (lane < nl) {
            const int nv = a ? nn[(size_t)q * nl + lane] : nc[(size_t)q * nl + lane];
            if (a) nc[(size_t)q * nl + lane] = nv;
            if (gather_next) nn2[(size_t)p2 * nl + lane] = nv;
        }
    }
    // this helper's partial sums; the last helper reduces them and resets the counters
    const FinishPart mine = block_sum_parts(e, (u128)dsum, na, s_w);
    if (threadIdx.x == 0) {
        parts[hb] = mine;
        __threadfence();
        last = atomicAdd(&tc->ticket, 1u) == nh - 1;
    }
    __syncthreads();
    if (!last) return;
    __threadfence();
    u128 E = 0, D = 0;
    unsigned A = 0;
    for (uint32_t j = threadIdx.x; j < nh; j += blockDim.x) {
        const unsigned long long* qq = reinterpret_cast<const unsigned long long*>(parts + j);
        E += ((u128)__ldcg(qq + 1) << 64) | __ldcg(qq + 0);
        D += ((u128)__ldcg(qq + 3) << 64) | __ldcg(qq + 2);
        A += (unsigned)__ldcg(qq + 4);
    }
    const FinishPart tot = block_sum_parts(E, D, A, s_w);
    for (uint32_t j = threadIdx.x; j < 64; j += blockDim.x) tc->dec[j] = 0;
    if (threadIdx.x == 0) {
        const u128 Et = ((u128)tot.e[1] << 64) | tot.e[0], Dd = ((u128)tot.d[1] << 64) | tot.d[0];
        const u128 Ea = Et + Dd;
        out->E_before[0] = tot.e[0];
        out->E_before[1] = tot.e[1];
        out->E_after[0] = (unsigned long long)Ea;
        out->E_after[1] = (unsigned long long)(Ea >> 64);
        out->dE_sum[0] = tot.d[0];
        out->dE_sum[1] = tot.d[1];
        out->accepted = tot.a / 2;
        if (check_prev && (__ldcg(&out[-1].E_after[0]) != tot.e[0] || __ldcg(&out[-1].E_after[1]) != tot.e[1]))
            atomicOr(err, 4);
        tc->com_next = 0;
        tc->ticket = 0;
    }
}

// Best-of-K REDRAW (K > 1, reading R19): one launch per colour class, one CTA per
// candidate pixel p of the class, step by step (the 4-Gram formulation of the K = 1 path would need
// (K+1)^2 window Grams).  The CTA stages p's current row and its K candidate rows in shared memory,
// each warp streams a share of the 224 neighbours' current rows (committed by the earlier classes)
// and forms the K+1 exact dot products per level with dp4a, every lane holding all of them after a
// butterfly; lane j < K accumulates dE_j = sum_l sum_o q(o, D(cn^j_p, c_q)) - q(o, D(c_p, c_q)) in
// int64 (R15).  The best candidate (lowest dE, ties to the lowest j, as the oracle) is accepted iff
// 2 dE < 0 and committed by the same CTA: members of a class are window-independent.
constexpr int KBEST_MAX = 8;
constexpr int KBEST_SPLIT = 4;  // CTAs per candidate (each sums a quarter of the window)
// grid (M, KBEST_SPLIT): CTA (m, sp) sums the neighbours w = sp, sp + KBEST_SPLIT, ... of candidate m
// into the exact int64 partials part[m][j] (integer atomics: order-independent); the last CTA of the
// candidate (ticket) decides, commits, and resets the partials and its ticket for the next class.
template <int R, int NV>
__global__ void __launch_bounds__(256) k_class_best(uint32_t s, uint32_t pass_t, uint64_t seed, uint32_t L, uint32_t K,
                                                    uint8_t* __restrict__ c, const uint8_t* __restrict__ cnK,
                                                    int* __restrict__ nc, const int* __restrict__ nnK,
                                                    uint2* __restrict__ U, const uint2* __restrict__ UnK,
                                                    uint32_t rowB, uint32_t Tp, uint32_t nl,
                                                    const double* __restrict__ W, LutArgs lut,
                                                    uint8_t* __restrict__ acc, i128* __restrict__ dEp,
                                                    uint8_t* __restrict__ log, int* __restrict__ err,
                                                    unsigned long long* __restrict__ part, unsigned int* __restrict__ tickets) {
    constexpr int WN = (2 * R + 1) * (2 * R + 1) - 1;
    extern __shared__ __align__(16) uint8_t xrows[];  // [K + 1][rowB]: c_p, cn^0_p .. cn^{K-1}_p
    __shared__ long long sdE[8][KBEST_MAX];
    __shared__ bool slast;
    const uint32_t M = (L / 8) * (L / 8), P = L * L, m = blockIdx.x, sp = blockIdx.y;
    const uint32_t p = class_pixel(L, seed, pass_t, s, m);
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarp = blockDim.x >> 5;
    const uint32_t n16 = rowB / 16;
    for (uint32_t j = threadIdx.x; j < (K + 1) * n16; j += blockDim.x) {
        const uint32_t v = j / n16, cidx = j - v * n16;
        const uint4* src = reinterpret_cast<const uint4*>(v == 0 ? c + (size_t)p * rowB
                                                                 : cnK + ((size_t)(v - 1) * P + p) * rowB);
        reinterpret_cast<uint4*>(xrows)[j] = src[cidx];
    }
    __syncthreads();
    const uint32_t x = p % L, y = p / L;
    long long dE = 0;  // lane j < K: candidate j's sum over this warp's neighbours
    for (uint32_t w = sp + KBEST_SPLIT * warp; w < (uint32_t)WN; w += KBEST_SPLIT * nwarp) {
        const int ww = w >= (uint32_t)(R * (2 * R + 1) + R) ? (int)w + 1 : (int)w;
        const int oy = ww / (2 * R + 1) - R, ox = ww % (2 * R + 1) - R;
        const uint32_t q = ((y + oy + L) & (L - 1)) * L + ((x + ox + L) & (L - 1));
        const double wt = W[w];
        const uint4* cq = reinterpret_cast<const uint4*>(c + (size_t)q * rowB);
        for (uint32_t l = 0; l < nl; ++l) {
            unsigned dot[NV];  // counts are unsigned bytes: dp4a.u32.u32
#pragma unroll
            for (int v = 0; v < NV; ++v) dot[v] = 0;
            for (uint32_t ci = l * (Tp / 16) + lane; ci < (l + 1) * (Tp / 16); ci += 32) {
                const uint4 b = __ldg(cq + ci);
#pragma unroll
                for (int v = 0; v < NV; ++v)
                    if (v <= (int)K) {
                        const uint4 a = reinterpret_cast<const uint4*>(xrows)[(size_t)v * n16 + ci];
                        dot[v] = __dp4a(a.x, b.x, dot[v]);
                        dot[v] = __dp4a(a.y, b.y, dot[v]);
                        dot[v] = __dp4a(a.z, b.z, dot[v]);
                        dot[v] = __dp4a(a.w, b.w, dot[v]);
                    }
            }
#pragma unroll
            for (int v = 0; v < NV; ++v)
#pragma unroll
                for (int o = 16; o; o >>= 1) dot[v] += __shfl_xor_sync(0xffffffffu, dot[v], o);
            const int nq = nc[(size_t)q * nl + l];
            const int D0 = nc[(size_t)p * nl + l] + nq - 2 * (int)dot[0];
            const int dm = lut.Dmax[l];
            if (lane < K) {
                int Dj = 0;
#pragma unroll
                for (int v = 1; v < NV; ++v)
                    if (v == (int)lane + 1) Dj = nnK[((size_t)lane * P + p) * nl + l] + nq - 2 * (int)dot[v];
                if ((unsigned)D0 > (unsigned)dm || (unsigned)Dj > (unsigned)dm) {
                    atomicOr(err, 1);
                } else {
                    dE += (long long)qterm(wt, lut.G[l], Dj) - (long long)qterm(wt, lut.G[l], D0);
                }
            }
        }
    }
    if (lane < K) sdE[warp][lane] = dE;
    __syncthreads();
    if (threadIdx.x < K) {
        long long t = 0;
        for (uint32_t wq = 0; wq < nwarp; ++wq) t += sdE[wq][threadIdx.x];
        atomicAdd(part + (size_t)m * KBEST_MAX + threadIdx.x, (unsigned long long)t);
    }
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) slast = atomicAdd(tickets + m, 1u) == KBEST_SPLIT - 1;
    __syncthreads();
    if (!slast) return;
    __threadfence();
    __shared__ int sbest;
    if (threadIdx.x == 0) {
        int best = -1;
        long long bv = 0;
        for (uint32_t j = 0; j < K; ++j) {
            const long long t = (long long)__ldcg(part + (size_t)m * KBEST_MAX + j);
            part[(size_t)m * KBEST_MAX + j] = 0;
            if (best < 0 || t < bv) {
                bv = t;
                best = (int)j;
            }
        }
        tickets[m] = 0;
        const i128 d = 2 * (i128)bv;
        const bool ok = d < 0;
        sbest = ok ? best : -1;
        acc[p] = ok;
        dEp[p] = ok ? d : (i128)0;
        if (log) log[(size_t)s * M + m] = ok;
    }
    __syncthreads();
    const int jb = sbest;
    if (jb < 0) return;
    const uint4* src = reinterpret_cast<const uint4*>(xrows) + (size_t)(jb + 1) * n16;
    uint4* dst = reinterpret_cast<uint4*>(c + (size_t)p * rowB);
    for (uint32_t j = threadIdx.x; j < n16; j += blockDim.x) dst[j] = src[j];
    if (threadIdx.x == 0) U[p] = UnK[(size_t)jb * P + p];
    if (threadIdx.x < nl) nc[(size_t)p * nl + threadIdx.x] = nnK[((size_t)jb * P + p) * nl + threadIdx.x];
}
// Pass sums of the best-of-K path: E_after = E_in + sum dEp (exact), accepted = sum acc.
__global__ void __launch_bounds__(1024) k_kstats(const i128* __restrict__ dEp, const uint8_t* __restrict__ acc,
                                                 uint32_t P, const unsigned long long* __restrict__ E_in,
                                                 PassStatsDev* __restrict__ out) {
    __shared__ FinishPart s_w[32];
    i128 d = 0;
    unsigned a = 0;
    for (uint32_t j = threadIdx.x; j < P; j += blockDim.x) {
        d += dEp[j];
        a += acc[j];
    }
    const FinishPart tot = block_sum_parts(0, (u128)d, a, s_w);
    if (threadIdx.x == 0) {
        const u128 E = ((u128)E_in[1] << 64) | E_in[0], D = ((u128)tot.d[1] << 64) | tot.d[0], Ea = E + D;
        out->E_before[0] = E_in[0];
        out->E_before[1] = E_in[1];
        out->E_after[0] = (unsigned long long)Ea;
        out->E_after[1] = (unsigned long long)(Ea >> 64);
        out->dE_sum[0] = tot.d[0];
        out->dE_sum[1] = tot.d[1];
        out->accepted = tot.a;
    }
}

// --------------------------------------------------------------------------- I_ref, readback
// Area of {(x,y) in [0,1]^2 : a(x - px) + b(y - py) >= 0}: the unit square clipped by the
// half-plane (walk the 4 edges, keep inside vertices and edge crossings), shoelace area. fp64.
__global__ void k_iref(const int2* __restrict__ ab, const uint2* __restrict__ pxy, uint32_t n, double* __restrict__ out) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double a = ab[i].x, b = ab[i].y;
    const double px = pxy[i].x * 0x1p-32, py = pxy[i].y * 0x1p-32;
    const double vx[4] = {0.0, 1.0, 1.0, 0.0}, vy[4] = {0.0, 0.0, 1.0, 1.0};
    double fx[8], fy[8];
    int n_out = 0;
    for (int e = 0; e < 4; ++e) {
        const int f = (e + 1) & 3;
        const double s0 = __dadd_rn(__dmul_rn(a, vx[e] - px), __dmul_rn(b, vy[e] - py));
        const double s1 = __dadd_rn(__dmul_rn(a, vx[f] - px), __dmul_rn(b, vy[f] - py));
        if (s0 >= 0) {
            fx[n_out] = vx[e];
            fy[n_out] = vy[e];
            ++n_out;
        }
        if ((s0 >= 0) != (s1 >= 0)) {
            const double t = s0 / (s0 - s1);
            fx[n_out] = __dadd_rn(vx[e], __dmul_rn(t, vx[f] - vx[e]));
            fy[n_out] = __dadd_rn(vy[e], __dmul_rn(t, vy[f] - vy[e]));
            ++n_out;
        }
    }
    double twice = 0.0;
    for (int j = 0; j < n_out; ++j) {
        const int k = (j + 1) % n_out;
        twice = __dadd_rn(twice, __dsub_rn(__dmul_rn(fx[j], fy[k]), __dmul_rn(fx[k], fy[j])));
    }
    out[i] = 0.5 * twice;
}

// cc component of Dt [l][p][H] (int4) -> int32 [l][p][H].
__global__ void k_dt_export(const int4* __restrict__ Dt, uint32_t P, uint32_t nl, int R, int* __restrict__ out) {
    const size_t H = (size_t)2 * R * R + 2 * R, HP = half_count_padded(R), n = (size_t)nl * P * H;
    const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const size_t lp = i / H;
    const int h = (int)(i - lp * H);
    const int oy = h < R ? 0 : 1 + (h - R) / (2 * R + 1), ox = h < R ? h + 1 : (h - R) % (2 * R + 1) - R;
    out[i] = reinterpret_cast<const int2*>(Dt)[lp * HP + hpad_index(ox, oy, R)].x;  // plane 0 .x = D(c_p, c_q)
}

// Internal [p][l][Tp] -> C-ABI [l][p][Ts].
__global__ void k_counts_export(const uint8_t* __restrict__ c, uint32_t P, uint32_t nl, uint32_t Tp, uint32_t Ts,
                                uint8_t* __restrict__ out) {
    const uint32_t lp = blockIdx.x, l = lp / P, p = lp - l * P;
    for (uint32_t i = threadIdx.x; i < Ts; i += blockDim.x)
        out[(size_t)lp * Ts + i] = c[((size_t)p * nl + l) * Tp + i];
}

// ------------------------------------------------------------- narrow count rows (f3)
// Per (level, integrand) offsets off[l][i] = round(N_l * I_ref,i) clamped to [0, N_l] (0 for the
// padding integrands); any integer offset keeps every distance exact, this one makes |delta| small
// (observed |c - N I_ref| <= 6 at N = 64).
__global__ void k_narrow_offsets(const double* __restrict__ iref, uint32_t Ts, uint32_t Tp, uint4 lo, uint4 hi,
                                 uint32_t nl, uint8_t* __restrict__ off) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= Tp) return;
    const uint32_t lv[8] = {lo.x, lo.y, lo.z, lo.w, hi.x, hi.y, hi.z, hi.w};
    for (uint32_t l = 0; l < nl; ++l) {
        long long o = 0;
        if (i < Ts) {
            o = __double2ll_rn((double)lv[l] * iref[i]);
            o = o < 0 ? 0 : o > (long long)lv[l] ? (long long)lv[l] : o;
        }
        off[(size_t)l * Tp + i] = (uint8_t)o;  // N_l <= 128
    }
}
// max over the tile of |c - off| per level -> rng[l].  Grid (blocks, nl): block (b, l) scans level l
// (16-byte chunks, grid-stride) keeping a per-byte running max (VABSDIFF4 / VMAX4), then one warp
// reduction and ONE atomicMax per block (a per-warp atomic on the single address rng[l] serialised
// 1M atomics for C5: 0.86 ms).
__global__ void __launch_bounds__(256) k_narrow_range(const uint8_t* __restrict__ c, uint32_t P, uint32_t Tp, uint32_t nl,
                                                      const uint8_t* __restrict__ off, int* __restrict__ rng) {
    const uint32_t l = blockIdx.y, g16 = Tp / 16;
    const size_t n = (size_t)P * g16;  // chunks of level l
    const uint4* cv4 = reinterpret_cast<const uint4*>(c);
    const uint4* ov4 = reinterpret_cast<const uint4*>(off + (size_t)l * Tp);
    uint32_t m = 0;  // four byte lanes
    for (size_t j = (size_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (size_t)gridDim.x * blockDim.x) {
        const size_t p = j / g16, g = j - p * g16;
        const uint4 cv = __ldcs(cv4 + (p * nl + l) * g16 + g);
        const uint4 ov = __ldg(ov4 + g);
        m = __vmaxu4(m, __vmaxu4(__vmaxu4(__vabsdiffu4(cv.x, ov.x), __vabsdiffu4(cv.y, ov.y)),
                                 __vmaxu4(__vabsdiffu4(cv.z, ov.z), __vabsdiffu4(cv.w, ov.w))));
    }
    unsigned mm = max(max(m & 0xffu, (m >> 8) & 0xffu), max((m >> 16) & 0xffu, m >> 24));
    mm = __reduce_max_sync(0xffffffffu, mm);
    __shared__ unsigned sm[8];
    if ((threadIdx.x & 31) == 0) sm[threadIdx.x >> 5] = mm;
    __syncthreads();
    if (threadIdx.x == 0) {
        for (uint32_t w = 1; w < (blockDim.x >> 5); ++w) mm = max(mm, sm[w]);
        if (mm) atomicMax(rng + l, (int)mm);
    }
}
// One thread per 16-integrand group (grid-stride); the row norms accumulate per warp in `norms`
// (zeroed before the launch) with one atomic per warp and row.
__global__ void __launch_bounds__(256) k_narrow_pack(const uint8_t* __restrict__ c, uint32_t P, uint32_t Tp, uint32_t nl,
                                                     const uint8_t* __restrict__ off, NarrowLayout lay, uint32_t rowBn,
                                                     uint8_t* __restrict__ out, int* __restrict__ norms) {
    const uint32_t g16 = Tp / 16, n = P * nl * g16;
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i - (threadIdx.x & 31) < n; i += gridDim.x * blockDim.x) {
        int nrm = 0;
        uint32_t row = 0;
        if (i < n) {
            row = i / g16;
            const uint32_t g = i - row * g16, p = row / nl, l = row - p * nl;
            const uint4 cv = __ldcs(reinterpret_cast<const uint4*>(c) + i);
            const uint32_t f = lay.fmt[l];
            const uint4 ov = f == BN_FMT_U8 ? make_uint4(0, 0, 0, 0) : __ldg(reinterpret_cast<const uint4*>(off + (size_t)l * Tp) + g);
            pack_chunk16(cv, ov, f, out + (size_t)p * rowBn + lay.lb[l], g, nrm);
        }
        if (g16 % 32 == 0) {  // the warp's 32 groups belong to one row
            nrm = (int)__reduce_add_sync(0xffffffffu, (unsigned)nrm);
            if ((threadIdx.x & 31) == 0 && i < n) atomicAdd(norms + row, nrm);
        } else if (i < n) {
            atomicAdd(norms + row, nrm);
        }
    }
}
// Inverse of k_narrow_pack: counts c = delta + off (u8 rows [p][l][Tp]) and their norms |c|^2.
__global__ void __launch_bounds__(256) k_narrow_unpack(const uint8_t* __restrict__ in, uint32_t P, uint32_t Tp, uint32_t nl,
                                                       const uint8_t* __restrict__ off, NarrowLayout lay, uint32_t rowBn,
                                                       uint8_t* __restrict__ c, int* __restrict__ norms) {
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t p = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (p >= P) return;
    for (uint32_t l = 0; l < nl; ++l) {
        uint8_t* row = c + ((size_t)p * nl + l) * Tp;
        const uint8_t* o = off + (size_t)l * Tp;
        const uint8_t* src = in + (size_t)p * rowBn + lay.lb[l];
        const uint32_t f = lay.fmt[l];
        int nrm = 0;
        for (uint32_t g = lane; g < Tp / 16; g += 32) {
            uint4 cv;
            uint8_t* cb = reinterpret_cast<uint8_t*>(&cv);
            if (f == BN_FMT_U8) {
                cv = *reinterpret_cast<const uint4*>(src + 16 * g);
            } else {
                const uint4 ov = *reinterpret_cast<const uint4*>(o + 16 * g);
                const uint8_t* ob = reinterpret_cast<const uint8_t*>(&ov);
                if (f == BN_FMT_E2M1) {
                    const uint2 w = *reinterpret_cast<const uint2*>(src + 8 * g);
#pragma unroll
                    for (int j = 0; j < 16; ++j)
                        cb[j] = (uint8_t)(dec_e2m1(((j < 8 ? w.x : w.y) >> (4 * (j & 7))) & 0xFu) + ob[j]);
                } else {
                    const uint32_t* s32 = reinterpret_cast<const uint32_t*>(src + 12 * g);
                    const unsigned long long lo = (unsigned long long)s32[0] | ((unsigned long long)s32[1] << 32);
                    const unsigned long long hi = s32[2];
#pragma unroll
                    for (int j = 0; j < 16; ++j) {
                        const int b = 6 * j;
                        unsigned long long e = b < 64 ? lo >> b : hi >> (b - 64);
                        if (b < 64 && b + 6 > 64) e |= hi << (64 - b);
                        cb[j] = (uint8_t)(dec_e3m2((uint32_t)e & 0x3Fu) + ob[j]);
                    }
                }
            }
            *reinterpret_cast<uint4*>(row + 16 * g) = cv;
#pragma unroll
            for (int j = 0; j < 16; ++j) nrm += (int)cb[j] * (int)cb[j];
        }
        nrm = (int)__reduce_add_sync(0xffffffffu, (unsigned)nrm);
        if (lane == 0) norms[(size_t)p * nl + l] = nrm;
    }
}

// Smooth evaluation integrands (§3.5 l.309-313): the estimate error of
// every (bump i, pixel p) at N samples, e = 1/N sum_k exp(-(x_k - cx)^2/(2 sx^2) - (y_k - cy)^2/(2 sy^2))
// - I_i, samples x_k = ((s^k.x + u_p.x) mod 2^32) 2^-32 in fp64; I_i host-built (erf products).
__global__ void __launch_bounds__(256) k_ev_smooth_err(const uint2* __restrict__ U, const uint2* __restrict__ S,
                                                       uint32_t N, const double4* __restrict__ bumps,
                                                       const double* __restrict__ ref, uint32_t nb, uint32_t P,
                                                       double* __restrict__ out) {
    const size_t t = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= (size_t)nb * P) return;
    const uint32_t i = (uint32_t)(t / P), p = (uint32_t)(t - (size_t)i * P);
    const double4 b = bumps[i];
    const double ax = 2.0 * b.z * b.z, ay = 2.0 * b.w * b.w;
    const uint2 u = U[p];
    double acc = 0.0;
    for (uint32_t k = 0; k < N; ++k) {
        const uint2 sk = S[k];
        const double x = (double)(sk.x + u.x) * 2.3283064365386963e-10, y = (double)(sk.y + u.y) * 2.3283064365386963e-10;
        acc += exp(-(x - b.x) * (x - b.x) / ax - (y - b.y) * (y - b.y) / ay);
    }
    out[t] = acc / (double)N - ref[i];
}

// Accept-log scatter is written directly by k_decide.

}  // namespace bn
