"""Seeded synthetic inputs shared by the oracle tests, the GPU tests and bench.py.

This module holds NO arithmetic of the method (no lattice, no counting, no energy, no
Philox of the optimiser): it only draws the *inputs* the paper leaves to the user --
the integrand bank ("randomly oriented Heavisides") and the initial tile
of shifts u_p (initialisation unstated, reading R16) -- and names the
five workload configurations of BASELINE.json.  Recipes are stated in DESIGN.md §4.

Bank recipe (reading R7): integer normal (a, b) uniform in [-2^15, 2^15)^2 conditioned on
2^20 <= a^2 + b^2 <= 2^30 (rejection => uniform direction); anchor (PX, PY) uniform uint32
(i.e. uniform in [0,1)^2 on the 2^-32 grid).  Tile recipe: u_p i.i.d. uniform uint32 pairs.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

#: Lattice direction vector d = (1, a) (reading R9): d1 = 1 satisfies the teaser's
#: d1 = 1 (mod 16) pin; a = 27 maximises the normalised minimum distance of the
#: 2^m-point prefixes for m = 4..7 among odd a < 256 (recorded, not from the paper).
D1, D2 = 1, 27


def make_bank(T: int, seed: int):
    """Integrand bank: (a, b) int32 [T], (px, py) uint32 [T].  Deterministic in (T, seed)."""
    if T < 1:
        raise ValueError("T must be >= 1")
    rng = np.random.Generator(np.random.PCG64(seed))
    a = np.empty(T, np.int32)
    b = np.empty(T, np.int32)
    n = 0
    while n < T:
        cand = rng.integers(-(1 << 15), 1 << 15, size=(2 * (T - n) + 8, 2), dtype=np.int64)
        r2 = cand[:, 0] ** 2 + cand[:, 1] ** 2
        ok = cand[(r2 >= (1 << 20)) & (r2 <= (1 << 30))]
        take = min(len(ok), T - n)
        a[n:n + take] = ok[:take, 0]
        b[n:n + take] = ok[:take, 1]
        n += take
    px = rng.integers(0, 1 << 32, size=T, dtype=np.uint64).astype(np.uint32)
    py = rng.integers(0, 1 << 32, size=T, dtype=np.uint64).astype(np.uint32)
    return a, b, px, py


def make_tile(L: int, seed: int) -> np.ndarray:
    """Initial tile u_p: uint32 [L*L, 2], i.i.d. uniform (SPEC.md l.280 reading)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    return rng.integers(0, 1 << 32, size=(L * L, 2), dtype=np.uint64).astype(np.uint32)


def make_permutation(P: int, seed: int) -> np.ndarray:
    """Precomputed permutation of the P pixel indices of the paper-verbatim optimiser
    ("we precompute a permutation of pixel indices that we store in a
    linear array"; how it is drawn is unstated -- uniform, reading R25).  uint32 [P]."""
    rng = np.random.Generator(np.random.PCG64(seed))
    return rng.permutation(P).astype(np.uint32)


def make_bumps(n: int, seed: int) -> np.ndarray:
    """Smooth (low-frequency) evaluation integrands, Gaussian bumps [n][4] = (cx, cy, sx, sy)
    (§3.5 l.309-313; evaluation only).  Reading R34: centres uniform in
    [0,1)^2, widths i.i.d. log-uniform in [0.05, 0.25]."""
    rng = np.random.Generator(np.random.PCG64(seed))
    c = rng.random((n, 2))
    w = np.exp(rng.uniform(np.log(0.05), np.log(0.25), size=(n, 2)))
    return np.ascontiguousarray(np.concatenate([c, w], axis=1), dtype=np.float64)


def axis_cut_bank(N: int, js, axis: str = "x"):
    """Lattice-aligned axis steps f = [x >= j/N] (or y): the exact-integral pin bank."""
    js = np.asarray(js, dtype=np.int64)
    T = len(js)
    a = np.zeros(T, np.int32)
    b = np.zeros(T, np.int32)
    px = np.zeros(T, np.uint32)
    py = np.zeros(T, np.uint32)
    cut = (js * (1 << 32) // N).astype(np.uint64).astype(np.uint32)
    if axis == "x":
        a[:] = 1
        px[:] = cut
    else:
        b[:] = 1
        py[:] = cut
    return a, b, px, py


@dataclass
class Config:
    """One of the five workloads of BASELINE.json['configs']."""

    name: str
    L: int
    levels: tuple
    T: int
    mode: int                 # 0 REDRAW, 1 SWAP
    passes: int
    pairs: int = 1            # independent dimension pairs (C4)
    seeds: tuple = (1, 2, 3)  # tile, bank, optimiser
    note: str = ""
    extra: dict = field(default_factory=dict)

    def pair_seeds(self, j: int):
        """Pair j uses every seed XOR j (reading R13)."""
        return tuple(s ^ j for s in self.seeds)


CONFIGS = {
    "C1": Config("C1", 16, (16,), 64, 0, 200,
                 note="16x16 tile, 2D rank-1 lattice, 16 spp, T=64 step integrands, 200 greedy passes"),
    "C2": Config("C2", 64, (4,), 256, 1, 100,
                 note="64x64 tile, 2D, 4 spp, T=256 integrands, swap-based optimisation, 1 GPU"),
    # C3, C4 and C5 run the SWAP (pixel-permuting) optimiser: the paper's own (PAPER.md l.228-229,
    # §3.4), and the one that lowers the denoised error (R32; REDRAW stays available,
    # bench.py --mode redraw)
    "C3": Config("C3", 128, (1, 4, 16, 64), 1024, 1, 100,
                 note="128x128 tile, 2D, 1/4/16/64 spp progressive, T=1024 integrands, 1 GPU"),
    "C4": Config("C4", 128, (16,), 1024, 1, 100, pairs=8,
                 note="128x128 tile, 8 independent dimension pairs (16D sampler), one pair per GPU"),
    "C5": Config("C5", 256, (16,), 8192, 1, 20,
                 note="256x256 tile, 2D, 16 spp, T=8192 integrands sharded across GPUs"),
}


def problem_inputs(cfg: Config, pair: int = 0):
    """(U, (a, b, px, py)) for pair `pair` of a config."""
    ts, bs, _ = cfg.pair_seeds(pair)
    return make_tile(cfg.L, ts), make_bank(cfg.T, bs)


def opt_seed(cfg: Config, pair: int = 0) -> int:
    return cfg.pair_seeds(pair)[2]
