/*
 * bn_oracle.c -- plain, slow, obviously-correct CPU ORACLE for the hot path of
 * Belcour & Heitz, "Lessons Learned and Improvements when Building Screen-Space
 * Samplers with Blue-Noise Error Distribution" (arXiv 2105.12620).
 *
 * THIS IS TEST INFRASTRUCTURE, NOT PRODUCT CODE.  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load it.  It shares no code,
 * header, table or constant generator with the CUDA path (paper_2105_12620_b200/csrc).
 *
 * Single-threaded C11, fp64 wherever floating point appears, compiled with
 * -O2 -ffp-contract=off.  Every function follows the paper (PAPER.md line numbers) or a
 * reading recorded in DESIGN.md §3 (R1..R16).  No blocking, no fusion, no caching of
 * intermediate tables: every distance is recomputed from the counts by its definition.
 *
 * Notation (§2 l.217-240, §3.2 l.258-266):
 *   s^k     = mod(Phi(k) * d, 1)          main sequence, rank-1 lattice   (l.260-261)
 *   s^k_p   = mod(s^k + u_p, 1)           toroidal-shift scrambling       (l.264-265, teaser l.54)
 *   I_p     = {1/N sum_k f_i(s^k_p)}      vector of test-integrand estimates (l.238-240)
 *   f_i     = randomly oriented Heaviside                                (l.239)
 *   E       = sum_p sum_{q in window} w(p-q) * exp(-||e_p - e_q|| / sigma_s^2)
 *             (north-star energy; Eq.1 l.232-237 supplies the spatial Gaussian 2.1^2)
 * Fixed point: every value in [0,1) is a uint32 U with value U / 2^32 (reading R15).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef __int128 i128;
typedef unsigned __int128 u128;

/* ------------------------------------------------------------------------------------------
 * Philox4x32-10 (Salmon et al., SC'11, "Parallel random numbers: as easy as 1, 2, 3").
 * The paper asks for a per-pass random scramble; the north star names
 * Philox keyed by pass/pixel.  Textbook definition; pinned by the Random123 known answers.
 * ---------------------------------------------------------------------------------------- */
void orc_philox4x32_10(const uint32_t ctr_in[4], const uint32_t key_in[2], uint32_t out[4]) {
    uint32_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
    uint32_t k0 = key_in[0], k1 = key_in[1];
    for (int round = 0; round < 10; ++round) {
        if (round > 0) {               /* key schedule: bump by the Weyl constants */
            k0 += 0x9E3779B9u;
            k1 += 0xBB67AE85u;
        }
        uint64_t p0 = (uint64_t)0xD2511F53u * (uint64_t)c0;
        uint64_t p1 = (uint64_t)0xCD9E8D57u * (uint64_t)c2;
        uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
        uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
        uint32_t n0 = hi1 ^ c1 ^ k0;
        uint32_t n1 = lo1;
        uint32_t n2 = hi0 ^ c3 ^ k1;
        uint32_t n3 = lo0;
        c0 = n0; c1 = n1; c2 = n2; c3 = n3;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* Philox keyed by the 64-bit seed: key = (seed lo, seed hi). */
static void philox_seed(uint64_t seed, uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3,
                        uint32_t out[4]) {
    uint32_t ctr[4] = {c0, c1, c2, c3};
    uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
    orc_philox4x32_10(ctr, key, out);
}

/* ------------------------------------------------------------------------------------------
 * Van der Corput radical inverse Phi(k) in base 2: the binary digits of
 * k mirrored about the binary point.  Returned as the 32-bit fixed-point numerator, i.e.
 * Phi(k) = orc_vdc_bits(k) / 2^32.  Written digit by digit, as the definition reads.
 * ---------------------------------------------------------------------------------------- */
uint32_t orc_vdc_bits(uint32_t k) {
    uint32_t r = 0;
    for (int bit = 0; bit < 32; ++bit) {
        if (k & (1u << bit)) r |= 1u << (31 - bit);   /* digit 2^bit -> 2^-(bit+1) */
    }
    return r;
}

/* Rank-1 lattice s^k = mod(Phi(k) * d, 1) with integer direction
 * vector d = (d1, d2) (reading R9).  In 32-bit fixed point, Phi(k)*d mod 1 is the product
 * of the numerator with d taken mod 2^32 -- exact, no rounding. xy[2k], xy[2k+1]. */
void orc_lattice(uint32_t d1, uint32_t d2, uint32_t n, uint32_t *xy) {
    for (uint32_t k = 0; k < n; ++k) {
        uint32_t phi = orc_vdc_bits(k);
        xy[2 * k + 0] = (uint32_t)((uint64_t)phi * d1);   /* mod 2^32 */
        xy[2 * k + 1] = (uint32_t)((uint64_t)phi * d2);
    }
}

/* Toroidal-shift scrambling K(s, u) = mod(s + u, 1). */
static uint32_t shift_mod1(uint32_t s, uint32_t u) { return (uint32_t)((uint64_t)s + u); }

/* Scrambled sample s^k_p = mod(s^k + u_p, 1) (teaser l.54), fixed point, out[0..1]. */
void orc_sample(uint32_t d1, uint32_t d2, uint32_t ux, uint32_t uy, uint32_t k, uint32_t out[2]) {
    uint32_t phi = orc_vdc_bits(k);
    out[0] = shift_mod1((uint32_t)((uint64_t)phi * d1), ux);
    out[1] = shift_mod1((uint32_t)((uint64_t)phi * d2), uy);
}

/* Heaviside test integrand f_i ("randomly oriented Heavisides"; reading R7/R8):
 *   f(x, y) = 1  iff  a*(x - px) + b*(y - py) >= 0,
 * evaluated exactly on the 32-bit grid: (X - PX) is the signed difference of two fixed-point
 * numbers (NOT wrapped -- the Heaviside lives on the unit square, not the torus). */
static int heaviside(int32_t a, int32_t b, uint32_t PX, uint32_t PY, uint32_t X, uint32_t Y) {
    int64_t dx = (int64_t)X - (int64_t)PX;
    int64_t dy = (int64_t)Y - (int64_t)PY;
    int64_t v = (int64_t)a * dx + (int64_t)b * dy;       /* |v| < 2^48, exact */
    return v >= 0;
}

typedef struct {
    uint32_t L;             /* tile side, pixels p = y*L + x                         */
    uint32_t T;             /* number of test integrands                              */
    uint32_t n_levels;      /* progressive spp levels (prefixes of the vdC order)     */
    uint32_t levels[8];     /* N_l, ascending powers of two <= 128                    */
    uint32_t d1, d2;        /* lattice direction vector                               */
    const int32_t *a, *b;   /* integrand normals   [T]                                */
    const uint32_t *px, *py;/* integrand anchors   [T], fixed point                   */
    double sigma_i;         /* spatial Gaussian, Eq.1: 2.1            */
    double sigma_s;         /* error-space scale (north star; reading R3)             */
    int32_t radius;         /* window radius R (reading R4)                           */
    int32_t form;           /* 0: north-star GF energy; 1: Eq. 1 as written; 2: Eq. 1  */
                            /* maximised (reading R1)                      */
} orc_problem;

/* Count c = #{k < N : f_i(s^k_p) = 1} (I_p,i = c / N).  Plain loop. */
uint32_t orc_count1(const orc_problem *pb, uint32_t ux, uint32_t uy, uint32_t i, uint32_t N) {
    uint32_t c = 0;
    for (uint32_t k = 0; k < N; ++k) {
        uint32_t s[2];
        orc_sample(pb->d1, pb->d2, ux, uy, k, s);
        c += (uint32_t)heaviside(pb->a[i], pb->b[i], pb->px[i], pb->py[i], s[0], s[1]);
    }
    return c;
}

/* Error-vector counts for every pixel: out[l][p][i] (level-major, as the C-ABI documents).
 * Same definition as orc_count1; the main sequence s^k is generated once (orc_lattice) and
 * each pixel's samples are its shift of it. */
void orc_counts(const orc_problem *pb, const uint32_t *U, uint32_t P, uint8_t *out) {
    const uint32_t Nmax = pb->levels[pb->n_levels - 1];
    uint32_t *S = malloc(sizeof(uint32_t) * 2 * Nmax);
    orc_lattice(pb->d1, pb->d2, Nmax, S);
    for (uint32_t l = 0; l < pb->n_levels; ++l)
        for (uint32_t p = 0; p < P; ++p)
            for (uint32_t i = 0; i < pb->T; ++i) {
                uint32_t c = 0;
                for (uint32_t k = 0; k < pb->levels[l]; ++k) {
                    uint32_t X = shift_mod1(S[2 * k], U[2 * p]), Y = shift_mod1(S[2 * k + 1], U[2 * p + 1]);
                    c += (uint32_t)heaviside(pb->a[i], pb->b[i], pb->px[i], pb->py[i], X, Y);
                }
                out[((size_t)l * P + p) * pb->T + i] = (uint8_t)c;
            }
    free(S);
}

/* Exact reference I_ref,i = area of {x in [0,1]^2 : a(x-px) + b(y-py) >= 0}
 * (teaser l.154 "I_ref"), by clipping the unit square against the
 * half-plane (Sutherland-Hodgman) and taking the shoelace area.  fp64. */
double orc_iref(int32_t a, int32_t b, uint32_t PX, uint32_t PY) {
    const double px = (double)PX / 4294967296.0, py = (double)PY / 4294967296.0;
    const double sq[4][2] = {{0, 0}, {1, 0}, {1, 1}, {0, 1}};
    double poly[8][2];
    int n = 0;
    for (int e = 0; e < 4; ++e) {
        const double *P0 = sq[e], *P1 = sq[(e + 1) % 4];
        double f0 = a * (P0[0] - px) + b * (P0[1] - py);
        double f1 = a * (P1[0] - px) + b * (P1[1] - py);
        if (f0 >= 0) { poly[n][0] = P0[0]; poly[n][1] = P0[1]; ++n; }
        if ((f0 >= 0) != (f1 >= 0)) {
            double t = f0 / (f0 - f1);
            poly[n][0] = P0[0] + t * (P1[0] - P0[0]);
            poly[n][1] = P0[1] + t * (P1[1] - P0[1]);
            ++n;
        }
    }
    double area2 = 0.0;
    for (int j = 0; j < n; ++j) {
        int k = (j + 1) % n;
        area2 += poly[j][0] * poly[k][1] - poly[k][0] * poly[j][1];
    }
    return 0.5 * area2;
}

/* ---------------------------------------------------------------------------------------
 * Energy (north star; Eq. 1 l.232-237 for the window weight; readings R1-R6, R15):
 *   w(o)   = exp(-|o|^2 / sigma_i^2)
 *   g_N(D) = exp(-(sqrt(D) / N) / sigma_s^2),   ||e_p - e_q|| = sqrt(D)/N exactly, because
 *            e = c/N - I_ref and I_ref cancels;  D = sum_i (c_p,i - c_q,i)^2  (integer)
 *   q(o,D) = round-to-nearest( 2^52 * (w(o) * g_N(D)) )           (uint64 fixed point, R15)
 *   E_fix  = sum_l sum_p sum_{o in O} q(o, D_l(p, p+o mod L))      (uint128, exact)
 * --------------------------------------------------------------------------------------- */
static double w_of(const orc_problem *pb, int ox, int oy) {
    return exp(-(double)(ox * ox + oy * oy) / (pb->sigma_i * pb->sigma_i));
}
static double g_of(const orc_problem *pb, uint64_t D, uint32_t N) {
    if (pb->form == 0) return exp(-(sqrt((double)D) / (double)N) / (pb->sigma_s * pb->sigma_s));
    /* Eq. 1: ||I_p - I_q||^2 = D / N^2 with I = c / N; divided by T so that the
     * fixed-point term w * g stays below 1.  Form 2 minimises 1 - that, i.e. maximises Eq. 1. */
    double sq = (double)D / (double)((uint64_t)N * N * pb->T);
    return pb->form == 1 ? sq : 1.0 - sq;
}
uint64_t orc_q(const orc_problem *pb, int ox, int oy, uint64_t D, uint32_t N) {
    double v = w_of(pb, ox, oy) * g_of(pb, D, N);
    return (uint64_t)nearbyint(ldexp(v, 52));
}

/* D_l(p,q) from two count rows of length T (the plain definition). */
static uint64_t dist2(const uint8_t *cp, const uint8_t *cq, uint32_t T) {
    uint64_t D = 0;
    for (uint32_t i = 0; i < T; ++i) {
        int64_t d = (int64_t)cp[i] - (int64_t)cq[i];
        D += (uint64_t)(d * d);
    }
    return D;
}

static uint32_t wrap(int64_t v, uint32_t L) { return (uint32_t)(((v % (int64_t)L) + L) % L); }

/* E over counts c[l][p][i]; Efix as (lo, hi) of a uint128 (E = Efix * 2^-52); Eplain: the same sum in fp64,
 * accumulated sequentially in raster x window order. */
void orc_energy(const orc_problem *pb, const uint8_t *c, uint64_t Efix[2], double *Eplain) {
    const uint32_t L = pb->L, P = L * L, T = pb->T;
    const int R = pb->radius;
    u128 E = 0;
    double Ep = 0.0;
    for (uint32_t l = 0; l < pb->n_levels; ++l) {
        const uint8_t *cl = c + (size_t)l * P * T;
        for (uint32_t y = 0; y < L; ++y)
            for (uint32_t x = 0; x < L; ++x)
                for (int oy = -R; oy <= R; ++oy)
                    for (int ox = -R; ox <= R; ++ox) {
                        if (ox == 0 && oy == 0) continue;
                        uint32_t qx = wrap((int64_t)x + ox, L), qy = wrap((int64_t)y + oy, L);
                        uint64_t D = dist2(cl + ((size_t)y * L + x) * T,
                                           cl + ((size_t)qy * L + qx) * T, T);
                        E += orc_q(pb, ox, oy, D, pb->levels[l]);
                        Ep += w_of(pb, ox, oy) * g_of(pb, D, pb->levels[l]);
                    }
    }
    Efix[0] = (uint64_t)E;
    Efix[1] = (uint64_t)(E >> 64);
    *Eplain = Ep;
}

/* ---------------------------------------------------------------------------------------
 * Energy change of replacing pixel p's count rows by new rows cn (all levels), against the
 * current counts c (north star "re-draws"; ordered pairs => factor 2, reading R6).
 *   dE = 2 * sum_l sum_{o in O} [ q(o, D(cn, c_{p+o})) - q(o, D(c_p, c_{p+o})) ]
 * 'skip' (a pixel index or UINT32_MAX) excludes one neighbour: used by SWAP for the partner.
 * --------------------------------------------------------------------------------------- */
static i128 delta_replace(const orc_problem *pb, const uint8_t *c, uint32_t p,
                          const uint8_t *cn /* [l][T] */, uint32_t skip) {
    const uint32_t L = pb->L, P = L * L, T = pb->T;
    const int R = pb->radius;
    const uint32_t x = p % L, y = p / L;
    i128 dE = 0;
    for (uint32_t l = 0; l < pb->n_levels; ++l) {
        const uint8_t *cl = c + (size_t)l * P * T;
        for (int oy = -R; oy <= R; ++oy)
            for (int ox = -R; ox <= R; ++ox) {
                if (ox == 0 && oy == 0) continue;
                uint32_t q = wrap((int64_t)y + oy, L) * L + wrap((int64_t)x + ox, L);
                if (q == skip) continue;
                uint64_t Dn = dist2(cn + (size_t)l * T, cl + (size_t)q * T, T);
                uint64_t Do = dist2(cl + (size_t)p * T, cl + (size_t)q * T, T);
                dE += (i128)orc_q(pb, ox, oy, Dn, pb->levels[l]);
                dE -= (i128)orc_q(pb, ox, oy, Do, pb->levels[l]);
            }
    }
    return 2 * dE;
}

/* Copy pixel p's rows (all levels) out of c[l][p][i]. */
static void get_rows(const orc_problem *pb, const uint8_t *c, uint32_t p, uint8_t *rows) {
    const uint32_t P = pb->L * pb->L, T = pb->T;
    for (uint32_t l = 0; l < pb->n_levels; ++l)
        memcpy(rows + (size_t)l * T, c + ((size_t)l * P + p) * T, T);
}
static void set_rows(const orc_problem *pb, uint8_t *c, uint32_t p, const uint8_t *rows) {
    const uint32_t P = pb->L * pb->L, T = pb->T;
    for (uint32_t l = 0; l < pb->n_levels; ++l)
        memcpy(c + ((size_t)l * P + p) * T, rows + (size_t)l * T, T);
}
static void rows_for_shift(const orc_problem *pb, uint32_t ux, uint32_t uy, uint8_t *rows) {
    for (uint32_t l = 0; l < pb->n_levels; ++l)
        for (uint32_t i = 0; i < pb->T; ++i)
            rows[(size_t)l * pb->T + i] = (uint8_t)orc_count1(pb, ux, uy, i, pb->levels[l]);
}

/* Brute-force pins: E after a single replacement minus E before, recomputed from scratch. */
void orc_delta_replace(const orc_problem *pb, const uint8_t *c, uint32_t p, uint32_t ux,
                       uint32_t uy, uint64_t dE[2]) {
    uint8_t *rows = malloc((size_t)pb->n_levels * pb->T);
    rows_for_shift(pb, ux, uy, rows);
    i128 d = delta_replace(pb, c, p, rows, UINT32_MAX);
    free(rows);
    dE[0] = (uint64_t)(u128)d;
    dE[1] = (uint64_t)((u128)d >> 64);
}

/* ---------------------------------------------------------------------------------------
 * Schedule of pass t (readings R10, R14; north star "graph-coloured pixel subsets, Philox
 * keyed by pass/pixel"; "XOR with a different seed per compute pass").
 * 64 colour steps s = 8r + k.  Orientation t&1 (0: lines are rows, 1: columns).
 *   A(t,r,k) = { (x,y) : y = 8b + r, x = 8a + ((delta(t,r,b) + k) & 7) }   (transposed if odd)
 *   delta(t,r,b) = Philox(seed; b, t, r, 2)[0] & 7,  active index m = b*(L/8) + a.
 * Members of one A are >= 8 > R apart (Chebyshev, on the torus): window-independent.
 * --------------------------------------------------------------------------------------- */
static uint32_t active_pixel(uint32_t L, uint64_t seed, uint32_t t, uint32_t r, uint32_t k,
                             uint32_t m) {
    uint32_t nb = L / 8, b = m / nb, a = m % nb, out[4];
    philox_seed(seed, b, t, r, 2, out);
    uint32_t along = 8 * a + ((out[0] + k) & 7), across = 8 * b + r;
    return (t & 1) ? along * L + across : across * L + along;
}

typedef struct {
    uint32_t mode;          /* 0 REDRAW, 1 SWAP                                       */
    uint32_t passes;
    uint32_t first_pass;    /* pass index t of the first pass (resume)                */
    uint32_t K;             /* re-draw candidates per pixel (best-of-K)               */
    uint64_t seed;
    uint32_t max_steps;     /* 0 = all 64; else stop each pass after this many steps  */
    uint32_t gauss_seidel;  /* 1: commit each accepted candidate immediately          */
    uint32_t energy_each_pass; /* 1: recompute E from scratch after every pass        */
} orc_opt;

typedef struct {
    uint32_t accepted, proposed;
    double E_plain;
    uint64_t E_fixed[2];
    uint64_t dE_sum[2];     /* sum of accepted dE (int128, two's complement)          */
} orc_stats;

/* Greedy independent-set optimisation (§3.4 l.291-302, north star):
 * every candidate of an active set is evaluated against the state before the step,
 * accepted iff dE < 0 (strict), and all accepted candidates are committed.
 * U: [2P] in/out; c: [l][P][T] in/out (must equal orc_counts(U) on entry).
 * accept_log: optional, [passes][64][M] bytes.  Returns 0 or -1 on bad arguments. */
int orc_optimize(const orc_problem *pb, uint32_t *U, uint8_t *c, const orc_opt *opt,
                 orc_stats *stats, uint8_t *accept_log) {
    const uint32_t L = pb->L, P = L * L, T = pb->T, nl = pb->n_levels;
    const uint32_t M = (L / 8) * (L / 8);
    const size_t rowlen = (size_t)nl * T;
    if (L < 16 || (L & (L - 1)) || pb->radius < 1 || pb->radius > 7) return -1;
    if (opt->mode > 1 || opt->K < 1 || (opt->mode == 1 && opt->K != 1)) return -1;
    uint8_t *cand = malloc(rowlen * M * opt->K);
    uint8_t *tmp = malloc(rowlen * 2);
    uint32_t *candU = malloc(sizeof(uint32_t) * 2 * M);
    uint32_t *partner = malloc(sizeof(uint32_t) * M);
    uint8_t *acc = malloc(M);
    i128 *dEs = malloc(sizeof(i128) * M);
    for (uint32_t pi = 0; pi < opt->passes; ++pi) {
        const uint32_t t = opt->first_pass + pi;
        uint32_t accepted = 0, proposed = 0;
        i128 dE_sum = 0;
        const uint32_t nsteps = opt->max_steps ? opt->max_steps : 64;
        for (uint32_t s = 0; s < nsteps; ++s) {
            const uint32_t r = s / 8, k = s % 8;
            memset(acc, 0, M);
            if (opt->mode == 0) {
                /* REDRAW: u'_j = Philox(seed; p, t, j, 1)[0..1], best of K, ties -> lowest j */
                for (uint32_t m = 0; m < M; ++m) {
                    uint32_t p = active_pixel(L, opt->seed, t, r, k, m);
                    i128 best = 0;
                    int bestj = -1;
                    for (uint32_t j = 0; j < opt->K; ++j) {
                        uint32_t o4[4];
                        philox_seed(opt->seed, p, t, j, 1, o4);
                        uint8_t *rows = cand + ((size_t)m * opt->K + j) * rowlen;
                        rows_for_shift(pb, o4[0], o4[1], rows);
                        i128 d = delta_replace(pb, c, p, rows, UINT32_MAX);
                        if (bestj < 0 || d < best) { best = d; bestj = j; }
                        if (bestj == (int)j) { candU[2 * m] = o4[0]; candU[2 * m + 1] = o4[1]; }
                    }
                    ++proposed;
                    dEs[m] = best;
                    partner[m] = (uint32_t)bestj;
                    if (best < 0) {
                        acc[m] = 1;
                        if (opt->gauss_seidel) {
                            set_rows(pb, c, p, cand + ((size_t)m * opt->K + bestj) * rowlen);
                            U[2 * p] = candU[2 * m]; U[2 * p + 1] = candU[2 * m + 1];
                        }
                    }
                }
                if (!opt->gauss_seidel)
                    for (uint32_t m = 0; m < M; ++m)
                        if (acc[m]) {
                            uint32_t p = active_pixel(L, opt->seed, t, r, k, m);
                            set_rows(pb, c, p, cand + ((size_t)m * opt->K + partner[m]) * rowlen);
                            U[2 * p] = candU[2 * m]; U[2 * p + 1] = candU[2 * m + 1];
                        }
            } else {
                /* SWAP: couples (m, m ^ kappa), kappa = 1 + Philox(seed; s, t, 0, 3)[0] mod (M-1) */
                uint32_t o4[4];
                philox_seed(opt->seed, s, t, 0, 3, o4);
                const uint32_t kappa = 1 + o4[0] % (M - 1);
                for (uint32_t m = 0; m < M; ++m) {
                    uint32_t mm = m ^ kappa;
                    if (mm < m) continue;
                    uint32_t p = active_pixel(L, opt->seed, t, r, k, m);
                    uint32_t q = active_pixel(L, opt->seed, t, r, k, mm);
                    uint8_t *rp = tmp, *rq = tmp + rowlen;
                    get_rows(pb, c, p, rp);
                    get_rows(pb, c, q, rq);
                    i128 d = delta_replace(pb, c, p, rq, q) + delta_replace(pb, c, q, rp, p);
                    ++proposed;
                    dEs[m] = d;
                    if (d < 0) {
                        acc[m] = 1;
                        if (opt->gauss_seidel) {
                            set_rows(pb, c, p, rq); set_rows(pb, c, q, rp);
                            uint32_t ux = U[2 * p], uy = U[2 * p + 1];
                            U[2 * p] = U[2 * q]; U[2 * p + 1] = U[2 * q + 1];
                            U[2 * q] = ux; U[2 * q + 1] = uy;
                        }
                    }
                }
                if (!opt->gauss_seidel)
                    for (uint32_t m = 0; m < M; ++m)
                        if (acc[m]) {
                            uint32_t p = active_pixel(L, opt->seed, t, r, k, m);
                            uint32_t q = active_pixel(L, opt->seed, t, r, k, m ^ kappa);
                            uint8_t *rp = tmp, *rq = tmp + rowlen;
                            get_rows(pb, c, p, rp); get_rows(pb, c, q, rq);
                            set_rows(pb, c, p, rq); set_rows(pb, c, q, rp);
                            uint32_t ux = U[2 * p], uy = U[2 * p + 1];
                            U[2 * p] = U[2 * q]; U[2 * p + 1] = U[2 * q + 1];
                            U[2 * q] = ux; U[2 * q + 1] = uy;
                        }
            }
            for (uint32_t m = 0; m < M; ++m)
                if (acc[m]) { ++accepted; dE_sum += dEs[m]; }
            if (accept_log) {
                /* log convention (include/bn.h): SWAP marks both members of an accepted couple */
                uint8_t *lg = accept_log + ((size_t)pi * 64 + s) * M;
                memcpy(lg, acc, M);
                if (opt->mode == 1) {
                    uint32_t o4[4];
                    philox_seed(opt->seed, s, t, 0, 3, o4);
                    const uint32_t kappa = 1 + o4[0] % (M - 1);
                    for (uint32_t m = 0; m < M; ++m)
                        if (acc[m]) lg[m ^ kappa] = 1;
                }
            }
        }
        if (stats) {
            stats[pi].accepted = accepted;
            stats[pi].proposed = proposed;
            stats[pi].dE_sum[0] = (uint64_t)(u128)dE_sum;
            stats[pi].dE_sum[1] = (uint64_t)((u128)dE_sum >> 64);
            if (opt->energy_each_pass) {
                orc_energy(pb, c, stats[pi].E_fixed, &stats[pi].E_plain);
            } else {
                stats[pi].E_fixed[0] = stats[pi].E_fixed[1] = 0;
                stats[pi].E_plain = 0.0;
            }
        }
    }
    free(cand); free(tmp); free(candU); free(partner); free(acc); free(dEs);
    return 0;
}

/* Pixel of active index m at step s of pass t (exposed so tests can check the schedule). */
uint32_t orc_active_pixel(uint32_t L, uint64_t seed, uint32_t t, uint32_t s, uint32_t m) {
    return active_pixel(L, seed, t, s / 8, s % 8, m);
}

/* ---------------------------------------------------------------------------------------
 * Paper-verbatim parallel optimisation (§3.4 l.291-307; SURVEY §8(f) row f1;
 * readings R11, R25-R27 in DESIGN.md §2).
 *
 * Couples of pass t (l.303-306: "we precompute a permutation of pixel indices that we store in
 * a linear array.  We scramble the pixel indices using an XOR with a different seed per
 * compute pass"):
 *   key(t)   = Philox(seed; t, 0, 0, 5)[0] & (P - 1)          (P a power of two: a bijection)
 *   sigma_j  = perm[j] ^ key(t)
 *   couple c = (sigma_2c, sigma_2c+1),   c < budget / 2       (l.298: budget N/4 pixels, R11)
 * Pixel-disjoint by construction (l.293-294 "a pixel in a swap couple is not used in another
 * couple").  Every couple is evaluated against the tile as it stands at the start of the pass
 * ("we evaluate the cost function with no modification", l.294-295; snapshot reading R26,
 * SPEC.md l.250), and every couple with dE < 0 is swapped.  Concurrent swaps of nearby
 * couples are not accounted for, so E may rise (l.295-297).
 * --------------------------------------------------------------------------------------- */
uint32_t orc_paper_key(uint64_t seed, uint32_t t, uint32_t P) {
    uint32_t o4[4];
    philox_seed(seed, t, 0, 0, 5, o4);
    return o4[0] & (P - 1);
}

/* Couples of one pass: out[2c], out[2c+1] for c < budget/2.  -1 if P is not a power of two
 * (the XOR would leave [0, P)) or the budget is odd / out of range. */
int orc_paper_couples(const uint32_t *perm, uint32_t P, uint32_t key, uint32_t budget,
                      uint32_t *out) {
    if (P == 0 || (P & (P - 1)) || (budget & 1) || budget > P || key >= P) return -1;
    for (uint32_t j = 0; j < budget; ++j) out[j] = perm[j] ^ key;
    return 0;
}

/* passes of the paper-verbatim optimiser.  perm: [P] permutation of pixel indices;
 * budget: pixels per pass (even, 2..P).  stats[pi]: accepted couples, proposed = budget/2,
 * dE_sum = sum of the accepted couples' snapshot dE, E after the pass recomputed from scratch.
 * accept_log: optional [passes][budget/2] bytes.  Returns 0, or -1 on bad arguments. */
int orc_paper_optimize(const orc_problem *pb, uint32_t *U, uint8_t *c, const uint32_t *perm,
                       uint32_t budget, uint32_t passes, uint32_t first_pass, uint64_t seed,
                       orc_stats *stats, uint8_t *accept_log) {
    const uint32_t L = pb->L, P = L * L, T = pb->T, nl = pb->n_levels;
    const size_t rowlen = (size_t)nl * T;
    if (L < 16 || (L & (L - 1)) || pb->radius < 1 || pb->radius > 7) return -1;
    if (budget < 2 || (budget & 1) || budget > P) return -1;
    uint8_t *seen = calloc(P, 1);
    for (uint32_t j = 0; j < P; ++j) {
        if (perm[j] >= P || seen[perm[j]]) { free(seen); return -1; }   /* not a permutation */
        seen[perm[j]] = 1;
    }
    free(seen);
    const uint32_t nc = budget / 2;
    uint32_t *pix = malloc(sizeof(uint32_t) * budget);
    i128 *dEs = malloc(sizeof(i128) * nc);
    uint8_t *rp = malloc(rowlen), *rq = malloc(rowlen);
    for (uint32_t pi = 0; pi < passes; ++pi) {
        const uint32_t t = first_pass + pi;
        orc_paper_couples(perm, P, orc_paper_key(seed, t, P), budget, pix);
        /* 1. every couple against the snapshot (the counts are not modified in this loop) */
        for (uint32_t k = 0; k < nc; ++k) {
            const uint32_t p = pix[2 * k], q = pix[2 * k + 1];
            get_rows(pb, c, p, rp);
            get_rows(pb, c, q, rq);
            dEs[k] = delta_replace(pb, c, p, rq, q) + delta_replace(pb, c, q, rp, p);
        }
        /* 2. swap every improving couple (disjoint: the order does not matter) */
        uint32_t accepted = 0;
        i128 dE_sum = 0;
        for (uint32_t k = 0; k < nc; ++k) {
            const int ok = dEs[k] < 0;
            if (accept_log) accept_log[(size_t)pi * nc + k] = (uint8_t)ok;
            if (!ok) continue;
            const uint32_t p = pix[2 * k], q = pix[2 * k + 1];
            get_rows(pb, c, p, rp);
            get_rows(pb, c, q, rq);
            set_rows(pb, c, p, rq);
            set_rows(pb, c, q, rp);
            uint32_t ux = U[2 * p], uy = U[2 * p + 1];
            U[2 * p] = U[2 * q]; U[2 * p + 1] = U[2 * q + 1];
            U[2 * q] = ux; U[2 * q + 1] = uy;
            ++accepted;
            dE_sum += dEs[k];
        }
        if (stats) {
            stats[pi].accepted = accepted;
            stats[pi].proposed = nc;
            stats[pi].dE_sum[0] = (uint64_t)(u128)dE_sum;
            stats[pi].dE_sum[1] = (uint64_t)((u128)dE_sum >> 64);
            orc_energy(pb, c, stats[pi].E_fixed, &stats[pi].E_plain);
        }
    }
    free(pix); free(dEs); free(rp); free(rq);
    return 0;
}

/* ---------------------------------------------------------------------------------------
 * Evaluation criterion (§3.3 l.270-284, teaser (c) l.154 "||(I_N (*) k_sigma) - I_ref||";
 * SURVEY §8 row f2; readings R29-R31 in DESIGN.md).  Plain definitions, O(P * taps) and O(P^2):
 *   e_i(p)    = c[l][p][i] / N_l - I_ref,i                     error image of integrand i
 *   k_sigma   = exp(-(dx^2 + dy^2) / (2 sigma^2)) on [-r, r]^2, r = ceil(4 sigma), / its sum
 *   rmse(s)   = 1/T sum_i sqrt( 1/P sum_p ( sum_d k_s(d) c[l][p+d][i]/N_l - I_ref,i )^2 )
 *               (toroidal: the tile repeats over the screen, so taps wrap
 *               mod L however large the kernel)
 *   S(f)      = 1/T sum_i | sum_p (e_i(p) - mean_i) exp(-2 pi i f.p / L) |^2   (DC = 0)
 *   profile_j = mean of S over the frequencies f (signed, |fx|,|fy| <= L/2) with
 *               floor(|f|) = j + 1, j = 0 .. L/2 - 1 (DC excluded)
 * --------------------------------------------------------------------------------------- */
static double gauss_unnormalised(double sigma, int r, double *k) {
    double Z = 0.0;
    for (int dy = -r; dy <= r; ++dy)
        for (int dx = -r; dx <= r; ++dx) {
            double v = exp(-(double)(dx * dx + dy * dy) / (2.0 * sigma * sigma));
            k[(dy + r) * (2 * r + 1) + (dx + r)] = v;
            Z += v;
        }
    return Z;
}

/* Normalised Gaussian kernel of radius ceil(4 sigma): k[(dy+r)(2r+1) + dx+r], returns r (or -1). */
int orc_gauss_kernel(double sigma, double *k, int kmax) {
    if (!(sigma > 0)) return -1;
    int r = (int)ceil(4.0 * sigma);
    if ((2 * r + 1) * (2 * r + 1) > kmax) return -1;
    double Z = gauss_unnormalised(sigma, r, k);
    for (int j = 0; j < (2 * r + 1) * (2 * r + 1); ++j) k[j] /= Z;
    return r;
}

int orc_denoised_rmse(const orc_problem *pb, const uint8_t *c, uint32_t l, const double *sigmas,
                      uint32_t n_sigmas, double *rmse) {
    const uint32_t L = pb->L, P = L * L, T = pb->T, N = pb->levels[l];
    if (l >= pb->n_levels) return -1;
    const uint8_t *cl = c + (size_t)l * P * T;
    for (uint32_t s = 0; s < n_sigmas; ++s) {
        int r = (int)ceil(4.0 * sigmas[s]);
        int kw = 2 * r + 1;
        double *k = malloc(sizeof(double) * kw * kw);
        if (orc_gauss_kernel(sigmas[s], k, kw * kw) < 0) { free(k); return -1; }
        double acc = 0.0;
        for (uint32_t i = 0; i < T; ++i) {
            const double ref = orc_iref(pb->a[i], pb->b[i], pb->px[i], pb->py[i]);
            double ss = 0.0;
            for (uint32_t y = 0; y < L; ++y)
                for (uint32_t x = 0; x < L; ++x) {
                    double v = 0.0;   /* (I_N (*) k_sigma)(p) */
                    for (int dy = -r; dy <= r; ++dy)
                        for (int dx = -r; dx <= r; ++dx) {
                            uint32_t q = wrap((int64_t)y + dy, L) * L + wrap((int64_t)x + dx, L);
                            v += k[(dy + r) * kw + (dx + r)] * ((double)cl[(size_t)q * T + i] / (double)N);
                        }
                    ss += (v - ref) * (v - ref);
                }
            acc += sqrt(ss / (double)P);
        }
        rmse[s] = acc / (double)T;
        free(k);
    }
    return 0;
}

int orc_error_spectrum(const orc_problem *pb, const uint8_t *c, uint32_t l, double *S /* [ky][kx] */,
                       double *profile /* [L/2] */) {
    const uint32_t L = pb->L, P = L * L, T = pb->T, N = pb->levels[l];
    if (l >= pb->n_levels) return -1;
    const uint8_t *cl = c + (size_t)l * P * T;
    const double two_pi = 6.283185307179586476925286766559;
    double *e = malloc(sizeof(double) * P);
    memset(S, 0, sizeof(double) * P);
    for (uint32_t i = 0; i < T; ++i) {
        const double ref = orc_iref(pb->a[i], pb->b[i], pb->px[i], pb->py[i]);
        double mean = 0.0;
        for (uint32_t p = 0; p < P; ++p) {
            e[p] = (double)cl[(size_t)p * T + i] / (double)N - ref;
            mean += e[p];
        }
        mean /= (double)P;
        for (uint32_t ky = 0; ky < L; ++ky)
            for (uint32_t kx = 0; kx < L; ++kx) {
                double re = 0.0, im = 0.0;
                for (uint32_t y = 0; y < L; ++y)
                    for (uint32_t x = 0; x < L; ++x) {
                        double ph = -two_pi * (double)((kx * x + ky * y) % L) / (double)L;
                        re += (e[y * L + x] - mean) * cos(ph);
                        im += (e[y * L + x] - mean) * sin(ph);
                    }
                S[ky * L + kx] += (re * re + im * im) / (double)T;
            }
    }
    free(e);
    if (profile) {
        double *sum = calloc(L / 2, sizeof(double));
        uint32_t *cnt = calloc(L / 2, sizeof(uint32_t));
        for (uint32_t ky = 0; ky < L; ++ky)
            for (uint32_t kx = 0; kx < L; ++kx) {
                int fx = kx <= L / 2 ? (int)kx : (int)kx - (int)L;
                int fy = ky <= L / 2 ? (int)ky : (int)ky - (int)L;
                int j = (int)floor(sqrt((double)(fx * fx + fy * fy)));
                if (j < 1 || j > (int)L / 2) continue;
                sum[j - 1] += S[ky * L + kx];
                cnt[j - 1] += 1;
            }
        for (uint32_t j = 0; j < L / 2; ++j) profile[j] = cnt[j] ? sum[j] / cnt[j] : 0.0;
        free(sum); free(cnt);
    }
    return 0;
}

/* ------------------------------------------------------------------------------------------
 * Smooth (low-frequency) test integrands -- evaluation only (§3.5
 * l.309-313 "achieves blue-noise distribution of integrand noise even for low frequency
 * integrands"; a Gaussian-bump family used only to EVALUATE a tile
 * optimised on Heavisides, with exact references by separable error-function products).
 *   f(x, y) = exp(-(x - cx)^2 / (2 sx^2) - (y - cy)^2 / (2 sy^2))      on [0,1)^2
 *   I       = X(cx, sx) X(cy, sy),  X(c, s) = s sqrt(pi/2) (erf((1 - c)/(s sqrt 2)) + erf(c/(s sqrt 2)))
 *   e_i(p)  = 1/N sum_{k<N} f_i(s^k_p) - I_i       (the pixel's estimate error, fp64)
 * bumps: [nb][4] = (cx, cy, sx, sy).
 * ---------------------------------------------------------------------------------------- */
static double erf_axis(double c, double s) {
    const double r2 = 1.4142135623730950488016887242097;
    return s * 1.2533141373155002512078826424055 * (erf((1.0 - c) / (s * r2)) + erf(c / (s * r2)));
}
double orc_bump_integral(double cx, double cy, double sx, double sy) { return erf_axis(cx, sx) * erf_axis(cy, sy); }

int orc_smooth_errors(const orc_problem *pb, const uint32_t *U, uint32_t l, uint32_t nb, const double *bumps,
                      double *e /* [nb][P] */) {
    const uint32_t L = pb->L, P = L * L;
    if (l >= pb->n_levels || nb == 0) return -1;
    const uint32_t N = pb->levels[l];
    for (uint32_t i = 0; i < nb; ++i) {
        const double cx = bumps[4 * i], cy = bumps[4 * i + 1], sx = bumps[4 * i + 2], sy = bumps[4 * i + 3];
        if (!(sx > 0) || !(sy > 0)) return -1;
        const double ref = orc_bump_integral(cx, cy, sx, sy);
        for (uint32_t p = 0; p < P; ++p) {
            double acc = 0.0;
            for (uint32_t k = 0; k < N; ++k) {
                uint32_t xy[2];
                orc_sample(pb->d1, pb->d2, U[2 * p], U[2 * p + 1], k, xy);
                const double x = (double)xy[0] / 4294967296.0, y = (double)xy[1] / 4294967296.0;
                acc += exp(-(x - cx) * (x - cx) / (2.0 * sx * sx) - (y - cy) * (y - cy) / (2.0 * sy * sy));
            }
            e[(size_t)i * P + p] = acc / (double)N - ref;
        }
    }
    return 0;
}

/* The evaluation criterion (§3.3) on error images e[ni][P] (same definitions as
 * orc_denoised_rmse / orc_error_spectrum, which form the images from counts). */
int orc_denoised_rmse_images(uint32_t L, uint32_t ni, const double *e, const double *sigmas, uint32_t n_sigmas,
                             double *rmse) {
    const uint32_t P = L * L;
    for (uint32_t s = 0; s < n_sigmas; ++s) {
        int r = (int)ceil(4.0 * sigmas[s]);
        int kw = 2 * r + 1;
        double *k = malloc(sizeof(double) * kw * kw);
        if (orc_gauss_kernel(sigmas[s], k, kw * kw) < 0) { free(k); return -1; }
        double acc = 0.0;
        for (uint32_t i = 0; i < ni; ++i) {
            double ss = 0.0;
            for (uint32_t y = 0; y < L; ++y)
                for (uint32_t x = 0; x < L; ++x) {
                    double v = 0.0;   /* (e (*) k_sigma)(p) */
                    for (int dy = -r; dy <= r; ++dy)
                        for (int dx = -r; dx <= r; ++dx) {
                            uint32_t q = wrap((int64_t)y + dy, L) * L + wrap((int64_t)x + dx, L);
                            v += k[(dy + r) * kw + (dx + r)] * e[(size_t)i * P + q];
                        }
                    ss += v * v;
                }
            acc += sqrt(ss / (double)P);
        }
        rmse[s] = acc / (double)ni;
        free(k);
    }
    return 0;
}

int orc_error_spectrum_images(uint32_t L, uint32_t ni, const double *e, double *S /* [ky][kx] */,
                              double *profile /* [L/2] or NULL */) {
    const uint32_t P = L * L;
    const double two_pi = 6.283185307179586476925286766559;
    memset(S, 0, sizeof(double) * P);
    for (uint32_t i = 0; i < ni; ++i) {
        const double *ei = e + (size_t)i * P;
        double mean = 0.0;
        for (uint32_t p = 0; p < P; ++p) mean += ei[p];
        mean /= (double)P;
        for (uint32_t ky = 0; ky < L; ++ky)
            for (uint32_t kx = 0; kx < L; ++kx) {
                double re = 0.0, im = 0.0;
                for (uint32_t y = 0; y < L; ++y)
                    for (uint32_t x = 0; x < L; ++x) {
                        double ph = -two_pi * (double)((kx * x + ky * y) % L) / (double)L;
                        re += (ei[y * L + x] - mean) * cos(ph);
                        im += (ei[y * L + x] - mean) * sin(ph);
                    }
                S[ky * L + kx] += (re * re + im * im) / (double)ni;
            }
    }
    if (profile) {
        double *sum = calloc(L / 2, sizeof(double));
        uint32_t *cnt = calloc(L / 2, sizeof(uint32_t));
        for (uint32_t ky = 0; ky < L; ++ky)
            for (uint32_t kx = 0; kx < L; ++kx) {
                int fx = kx <= L / 2 ? (int)kx : (int)kx - (int)L;
                int fy = ky <= L / 2 ? (int)ky : (int)ky - (int)L;
                int j = (int)floor(sqrt((double)(fx * fx + fy * fy)));
                if (j < 1 || j > (int)L / 2) continue;
                sum[j - 1] += S[ky * L + kx];
                cnt[j - 1] += 1;
            }
        for (uint32_t j = 0; j < L / 2; ++j) profile[j] = cnt[j] ? sum[j] / cnt[j] : 0.0;
        free(sum); free(cnt);
    }
    return 0;
}
