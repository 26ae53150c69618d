/*
 * bn.h -- C-ABI of the B200-native blue-noise screen-space sampler optimiser
 * (Belcour & Heitz, arXiv 2105.12620; hot path = north star of BASELINE.json).
 *
 * The library (paper_2105_12620_b200/libbn.so) owns all device state of ONE tile problem
 * ("context"): the u_p tile, the integer error-vector counts, the energy look-up tables and
 * the per-pass work buffers.  Every step of the hot path runs in hand-written sm_100a
 * kernels; there is no CPU fallback.
 *
 * Conventions
 *  - Fixed point: a value v in [0,1) is the uint32 V with v = V / 2^32.
 *  - Pixels: p = y * L + x, 0 <= x, y < L; the tile repeats toroidally.
 *  - Tiles:  u_xy[2p + 0] = u_p.x, u_xy[2p + 1] = u_p.y                (uint32, 8 B / pixel)
 *  - Counts: out[(l * P + p) * Ts + i] = c_l,p,i = #{k < N_l : f_i(mod(s^k + u_p, 1)) = 1}
 *            (uint8, level-major; Ts = t_end - t_begin of this context's bank shard).
 *            The error vector of PAPER.md l.238-240 is e_p,i = c / N_l - I_ref,i exactly.
 *  - Ownership: the caller owns every buffer passed in or out; inputs are copied during the
 *    call.  Device pointers (is_device != 0) must be device memory of the context's device
 *    (e.g. torch tensor data_ptr()).
 *  - Streams: calls are enqueued on the context's stream.  Calls that return host data
 *    (bn_energy, bn_optimize with stats/accept_log, host get_tile/eval_counts,
 *    bn_get_references) synchronise that stream before returning.
 *  - Errors: every int-returning call returns a status below; bn_last_error() returns a
 *    human-readable message for the last failure on that context.  A failed call leaves the
 *    context's previously committed state unchanged unless it reports BN_ECUDA.
 *  - Threading: a context is single-stream and not thread-safe; distinct contexts are
 *    independent (one per GPU, rank or dimension pair).
 */
#ifndef BN_H
#define BN_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum bn_status {
    BN_OK = 0,
    BN_EINVAL = 1, /* argument outside the documented domain                            */
    BN_ECUDA = 2,  /* CUDA runtime / launch failure (message has cudaGetErrorString)     */
    BN_ENCCL = 3,  /* NCCL failure (multi-GPU bank sharding)                             */
    BN_ENOMEM = 4, /* device allocation failed                                          */
    BN_ESTATE = 5  /* call order violated, or an internal invariant failed              */
};

typedef struct bn_ctx bn_ctx;

/* Create a context on CUDA device `cuda_device`, enqueuing work on `cuda_stream`
 * (a cudaStream_t cast to uintptr_t; 0 = the legacy default stream).  *out = NULL on error. */
int bn_create(bn_ctx **out, int cuda_device, uintptr_t cuda_stream);
void bn_destroy(bn_ctx *ctx);
const char *bn_last_error(const bn_ctx *ctx);
/* Library build string (arch, version); never NULL. */
const char *bn_version(void);

/* Main sequence s^k = mod(Phi(k) d, 1) (§3.2 l.258-263): rank-1 lattice with
 * integer direction vector d = (d1, d2), van der Corput order.  spp_levels[0..n_levels) are
 * the progressive sample counts N_l (prefixes of the vdC order): strictly ascending powers
 * of two in [1, 128], 1 <= n_levels <= 8.  EINVAL otherwise. */
int bn_set_lattice(bn_ctx *ctx, uint32_t d1, uint32_t d2, const uint32_t *spp_levels,
                   uint32_t n_levels);

/* Bank of T Heaviside test integrands ("randomly oriented Heavisides"):
 *   f_i(x, y) = 1  iff  a_i (x - px_i) + b_i (y - py_i) >= 0   (exact on the 2^-32 grid)
 * a, b: int32 [T] with |a|, |b| <= 2^15 (so the test is exact in int64); px, py: uint32 [T]
 * fixed-point anchors.  Host arrays, copied.  This context evaluates the shard
 * [t_begin, t_end) (0 <= t_begin < t_end <= T); the energy always uses the full-T distance
 * (shards are summed across ranks by bn_comm_init's communicator).  EINVAL on T = 0,
 * bad range or |a|,|b| too large. */
int bn_set_bank(bn_ctx *ctx, uint32_t T, const int32_t *a, const int32_t *b,
                const uint32_t *px, const uint32_t *py, uint32_t t_begin, uint32_t t_end);

/* Exact references I_ref,i (area of the half-plane inside [0,1]^2; teaser l.154) of this
 * context's shard, fp64, written to host iref[t_end - t_begin].  Computed on the device. */
int bn_get_references(bn_ctx *ctx, double *iref);

/* Blue-noise energy parameters (north star; Eq. 1 PAPER.md l.232-237 for sigma_i = 2.1):
 *   E = sum_l sum_p sum_{o in O} q(o, D_l(p, p+o)),   O = [-R,R]^2 \ {0} (toroidal),
 *   q(o, D) = rn_uint64( 2^52 * exp(-|o|^2 / sigma_i^2) * exp(-(sqrt(D)/N_l) / sigma_s^2) )
 *   D_l(p,q) = sum_i (c_l,p,i - c_l,q,i)^2 = N_l^2 ||e_p - e_q||^2   (exact integer)
 * Defaults 2.1, 1.0, 7.  radius in [1, 7] (the stride-8 colouring needs R < 8); sigmas > 0. */
int bn_set_energy(bn_ctx *ctx, double sigma_i, double sigma_s, int32_t radius);

/* Energy form (reading R1): which g(D) the energy above uses.
 *   BN_E_GF      g = exp(-(sqrt(D)/N_l) / sigma_s^2)   north-star Georgiev-Fajardo form (default)
 *   BN_E_EQ1     g = D / (N_l^2 T) = ||I_p - I_q||^2 / T   Eq. 1 literally,
 *                minimised ("reduce the following loss"); the 1/T keeps w*g < 1 for the fixed point
 *   BN_E_EQ1_MAX g = 1 - D / (N_l^2 T): minimising it maximises Eq. 1 (the blue-noise direction)
 * sigma_s is ignored by the Eq. 1 forms.  EINVAL on an unknown form. */
enum bn_energy_form { BN_E_GF = 0, BN_E_EQ1 = 1, BN_E_EQ1_MAX = 2 };
int bn_set_energy_form(bn_ctx *ctx, uint32_t form);

/* Load the tile U (L*L pixels, L a power of two in [16, 2048], L > 2R) and build its counts.
 * u_xy: [2 L L] uint32, host (is_device = 0) or device.  Requires lattice and bank.
 * Returns once a host u_xy has been copied (it may then be reused); the counts are built
 * asynchronously on the context's stream, ordered before every later call on it. */
int bn_set_tile(bn_ctx *ctx, uint32_t L, const uint32_t *u_xy, int is_device);
/* Copy the current tile out ([2 L L] uint32) to host or device memory. */
int bn_get_tile(bn_ctx *ctx, uint32_t *u_xy, int is_device);

/* Exact error-vector representation: the counts of the current tile, layout in the header
 * comment, n_levels * L*L * (t_end - t_begin) bytes, host or device. */
int bn_eval_counts(bn_ctx *ctx, uint8_t *out, int is_device);

/* Energy of the current tile, recomputed from the counts (not incremental).
 * E_fixed[0..1] = (low, high) 64-bit words of the exact uint128 sum; *E = E_fixed * 2^-52.
 * Either pointer may be NULL.  Multi-GPU: collective over the communicator. */
int bn_energy(bn_ctx *ctx, double *E, uint64_t E_fixed[2]);

enum bn_mode { BN_REDRAW = 0, BN_SWAP = 1, BN_PAPER_SWAP = 2 };

typedef struct {
    uint32_t mode;       /* BN_REDRAW: re-draw u_p; BN_SWAP: swap u_p within couples;        */
                         /* BN_PAPER_SWAP: the paper's snapshot couples (bn_set_permutation) */
    uint32_t passes;     /* number of passes to run                                       */
    uint32_t first_pass; /* pass index t of the first pass (resume = continue counting)   */
    uint32_t K;          /* re-draw candidates per pixel: 1, or 2..8 for best-of-K REDRAW  */
    uint64_t seed;       /* Philox4x32-10 key of the optimiser                             */
    uint32_t budget;     /* BN_PAPER_SWAP: pixels per pass (even, 2..L*L; 0 = L*L/4, the     */
                         /* paper's N/4); ignored by the other modes         */
    uint32_t reserved;   /* must be 0                                                       */
} bn_opt_params;

typedef struct {
    uint32_t accepted;   /* candidates (REDRAW) or couples (SWAP, PAPER_SWAP) accepted      */
    uint32_t proposed;   /* candidates (= L*L), couples (= L*L/2) or budget/2 evaluated    */
    double E;            /* E_fixed * 2^-52 after the pass                                */
    uint64_t E_fixed[2]; /* exact energy after the pass (uint128, low word first)          */
    uint64_t dE_sum[2];  /* exact sum of the accepted dE (int128, two's complement)        */
} bn_pass_stats;

/* Run `passes` optimisation passes (§3.4 l.291-302; north star):
 * pass t visits the 64 colour classes s = 8r + k of the stride-8 schedule
 *   A(t,r,k) = {(x,y): y = 8b + r, x = 8a + ((delta(t,r,b) + k) & 7)}  (transposed for odd t),
 *   delta(t,r,b) = Philox(seed; b, t, r, 2)[0] & 7,  active index m = b (L/8) + a,
 * in order; every member of a class is window-independent of the others.  REDRAW proposes
 * u'_p = Philox(seed; p, t, 0, 1)[0..1]; SWAP couples m with m ^ kappa,
 * kappa = 1 + Philox(seed; s, t, 0, 3)[0] mod (M - 1), M = (L/8)^2.  A candidate (couple) is
 * accepted iff its exact dE < 0 against the state left by the earlier classes.
 * stats: host [passes] or NULL.  accept_log: host [passes][64][M] bytes (1 = accepted, SWAP:
 * both members of an accepted couple) or NULL.  EINVAL on an unknown mode, K outside [1, 8] or
 * K > 1 with a mode other than BN_REDRAW.
 *
 * Best-of-K REDRAW (K > 1): pixel p of class s draws K candidates
 * u'_j = Philox(seed; p, t, j, 1)[0..1], j < K, takes the one with the lowest exact dE against the
 * state left by the earlier classes (ties to the lowest j) and accepts it iff dE < 0.  Runs step by
 * step (one launch per class); single-GPU only (EINVAL with a communicator).
 *
 * BN_PAPER_SWAP (§3.4 l.291-307 verbatim): pass t forms the couples
 *   c = (perm[2c] ^ key(t), perm[2c+1] ^ key(t)),  c < budget/2,
 *   key(t) = Philox(seed; t, 0, 0, 5)[0] & (L*L - 1)   ("XOR with a different seed per pass"),
 * from the permutation given to bn_set_permutation; every couple's swap dE is evaluated against
 * the tile at the start of the pass and every couple with dE < 0 is swapped.  Concurrent swaps
 * of nearby couples are not accounted for, so E may rise (l.295-297): stats[].E is the energy
 * recomputed after the pass (one extra energy evaluation after the last pass), dE_sum the sum of
 * the accepted couples' snapshot dE.  accept_log[pass][c] = couple c's flag (first budget/2
 * bytes of each pass's 64*M).  ESTATE if no permutation of L*L entries is set; EINVAL on a
 * bad budget. */
int bn_optimize(bn_ctx *ctx, const bn_opt_params *params, bn_pass_stats *stats,
                uint8_t *accept_log);

/* Synchronise the context's stream and report the device invariant flag: every launch since the
 * flag was last read ORs into it (window distance outside [0, T N_l^2]; an exact dE term outside
 * +-2^55 (reading R15); a pass whose recomputed start energy differs from the previous pass's
 * E + sum dE).  bn_optimize with stats/accept_log and bn_energy read it too; reading clears it.
 * BN_OK if clean, BN_ESTATE (message in bn_last_error) if an invariant failed. */
int bn_check(bn_ctx *ctx);

/* Evaluation criterion (§3.3 l.270-284, teaser (c) "||(I_N (*) k_sigma) - I_ref||";
 * SURVEY §8 f2) of the current tile at progressive level `level`, over this context's integrand
 * shard [t_begin, t_end) (Ts integrands), error images e_i(p) = c_l,p,i / N_l - I_ref,i:
 *   rmse[s]   = 1/Ts sum_i sqrt( 1/P sum_p ((k_s (*) e_i)(p))^2 ),  s < n_sigmas (<= 64), with
 *               k_s the Gaussian exp(-(dx^2+dy^2)/(2 sigma_s^2)), |dx|,|dy| <= ceil(4 sigma_s),
 *               normalised to sum 1 and applied toroidally (the tile repeats; taps wrap mod L)
 *   spectrum  [L*L] (index ky*L + kx, DC first) = 1/Ts sum_i |DFT(e_i - mean e_i)|^2, or NULL
 *   profile   [L/2]: mean of the spectrum over the frequencies with floor(|f|) = j + 1 (signed
 *               frequencies, DC excluded), or NULL
 * fp64, through the 2D DFT of every error image (Parseval); host outputs; synchronises.
 * EINVAL on level >= n_levels, a sigma outside (0, 1e4], n_sigmas > 64 or L > 256. */
int bn_eval_quality(bn_ctx *ctx, uint32_t level, const double *sigmas, uint32_t n_sigmas,
                    double *rmse, double *spectrum, double *profile);

/* The same criterion for the smooth (low-frequency) evaluation integrands (§3.5
 * l.309-313 "blue-noise distribution of integrand noise even for low frequency integrands";
 * SURVEY §8 f4; used to evaluate a tile optimised on Heavisides, never to optimise):
 *   f_i(x, y) = exp(-(x - cx)^2 / (2 sx^2) - (y - cy)^2 / (2 sy^2)),  bumps [n_bumps][4] = (cx, cy, sx, sy)
 *   e_i(p)    = 1/N_l sum_{k < N_l} f_i(s^k_p) - I_i   (fp64 at the tile's samples),
 *   I_i       = the exact integral over [0,1]^2 (separable erf product, host libm), also returned
 *               in iref [n_bumps] if non-NULL;
 * rmse / spectrum / profile as bn_eval_quality over the n_bumps error images.  Host outputs;
 * synchronises.  EINVAL on level >= n_levels, no bumps, a width <= 0 or not finite, bad sigmas or
 * L > 256. */
int bn_eval_smooth(bn_ctx *ctx, uint32_t level, uint32_t n_bumps, const double *bumps, const double *sigmas,
                   uint32_t n_sigmas, double *rmse, double *spectrum, double *profile, double *iref);

/* Precomputed permutation of the pixel indices used by BN_PAPER_SWAP (PAPER.md l.303-304:
 * "we precompute a permutation of pixel indices that we store in a linear array").
 * perm: host uint32 [n], n = L*L of the tile the optimiser will run on, every index in [0, n)
 * exactly once (EINVAL otherwise).  Copied. */
int bn_set_permutation(bn_ctx *ctx, const uint32_t *perm, uint32_t n);

/* Window distances of the current tile over THIS context's bank shard (no cross-rank sum):
 * out[(l * P + p) * H + h] = D_l(p, p + o_h) restricted to integrands [t_begin, t_end),
 * h indexing the half window {o: oy > 0 or (oy == 0 and ox > 0)} ordered oy = 0, ox = 1..R, then
 * oy = 1..R, ox = -R..R (H = 2R^2 + 2R).  int32, host or device.  Summing the outputs of the
 * shards of a bank gives the full-bank distances exactly (the multi-GPU decomposition). */
int bn_window_distances(bn_ctx *ctx, int32_t *out, int is_device);

/* Multi-GPU bank sharding: join an NCCL communicator (ncclUniqueId bytes, 128 B, from rank 0
 * via torch.distributed) of `world` ranks, one context per rank, every rank holding the same
 * tile and its own [t_begin, t_end) shard.  The only exchange is an int32 sum over ranks of
 * the partial window distances, once per pass.  ENCCL on failure. */
int bn_comm_init(bn_ctx *ctx, const void *nccl_unique_id, int rank, int world);
/* Size of ncclUniqueId (128) and a fresh id for rank 0 to broadcast. */
int bn_comm_unique_id(void *out128);

/* Kernel launches this context has issued since creation (for the bench's gpu_launches). */
uint64_t bn_launch_count(const bn_ctx *ctx);

/* Per-kernel device time, measured with CUDA events recorded on the context's stream around
 * every launch while enabled (the bench's roofline line).  bn_profile_enable(ctx, 1) clears
 * and starts accumulation, 0 stops it.  bn_profile_get synchronises the stream and returns the
 * summed milliseconds and launch count of one kernel class. */
enum bn_kernel_id {
    BN_K_COUNTS = 0, /* candidate / tile error-vector counts          */
    BN_K_GATHER = 1, /* SWAP candidate gather                         */
    BN_K_GRAM = 2,   /* windowed distances (4 per neighbour pair)     */
    BN_K_LUT = 3,    /* fixed-point energy terms, dE tables, E        */
    BN_K_DECIDE = 4, /* colour-class decisions                        */
    BN_K_STATS = 5,  /* exact per-pass reductions                     */
    BN_K_COMMIT = 6, /* commit accepted rows / shifts                 */
    BN_K_TAIL = 7,   /* fused pass tail: decisions + commit / next gather (SWAP, 64 <= L <= 128) */
    BN_K_COUNT_IDS = 8
};
int bn_profile_enable(bn_ctx *ctx, int enable);
int bn_profile_get(bn_ctx *ctx, uint32_t kernel_id, double *total_ms, uint64_t *launches);

#ifdef __cplusplus
}
#endif
#endif /* BN_H */
