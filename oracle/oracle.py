"""ctypes wrapper around the plain CPU oracle ``oracle/bn_oracle.c``.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this module.  The product path
(``paper_2105_12620_b200``) never imports it, and it imports nothing from the product.

Every function documents the PAPER.md passage it follows; see the C source for the
arithmetic.  Arrays are numpy; layouts match the C-ABI documentation in ``include/bn.h``
(counts ``[level][pixel][integrand]``, tiles ``[pixel][2]`` uint32 fixed point).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "bn_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

# -ffp-contract=off: no fused multiply-add may change fp64 rounding (reading R15).
CFLAGS = ["-O2", "-std=gnu11", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared"]


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (it is a checker, built but never used by the product)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", *CFLAGS, "-o", _LIB, _SRC, "-lm"])
    return _LIB


class Problem(ctypes.Structure):
    _fields_ = [
        ("L", ctypes.c_uint32),
        ("T", ctypes.c_uint32),
        ("n_levels", ctypes.c_uint32),
        ("levels", ctypes.c_uint32 * 8),
        ("d1", ctypes.c_uint32),
        ("d2", ctypes.c_uint32),
        ("a", ctypes.c_void_p),
        ("b", ctypes.c_void_p),
        ("px", ctypes.c_void_p),
        ("py", ctypes.c_void_p),
        ("sigma_i", ctypes.c_double),
        ("sigma_s", ctypes.c_double),
        ("radius", ctypes.c_int32),
        ("form", ctypes.c_int32),
    ]


class Opt(ctypes.Structure):
    _fields_ = [
        ("mode", ctypes.c_uint32),
        ("passes", ctypes.c_uint32),
        ("first_pass", ctypes.c_uint32),
        ("K", ctypes.c_uint32),
        ("seed", ctypes.c_uint64),
        ("max_steps", ctypes.c_uint32),
        ("gauss_seidel", ctypes.c_uint32),
        ("energy_each_pass", ctypes.c_uint32),
    ]


class Stats(ctypes.Structure):
    _fields_ = [
        ("accepted", ctypes.c_uint32),
        ("proposed", ctypes.c_uint32),
        ("E_plain", ctypes.c_double),
        ("E_fixed", ctypes.c_uint64 * 2),
        ("dE_sum", ctypes.c_uint64 * 2),
    ]


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        P = ctypes.POINTER
        _lib.orc_philox4x32_10.argtypes = [P(ctypes.c_uint32), P(ctypes.c_uint32), P(ctypes.c_uint32)]
        _lib.orc_vdc_bits.argtypes = [ctypes.c_uint32]
        _lib.orc_vdc_bits.restype = ctypes.c_uint32
        _lib.orc_lattice.argtypes = [ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_void_p]
        _lib.orc_sample.argtypes = [ctypes.c_uint32] * 5 + [P(ctypes.c_uint32)]
        _lib.orc_iref.argtypes = [ctypes.c_int32, ctypes.c_int32, ctypes.c_uint32, ctypes.c_uint32]
        _lib.orc_iref.restype = ctypes.c_double
        _lib.orc_count1.argtypes = [P(Problem), ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint32]
        _lib.orc_count1.restype = ctypes.c_uint32
        _lib.orc_counts.argtypes = [P(Problem), ctypes.c_void_p, ctypes.c_uint32, ctypes.c_void_p]
        _lib.orc_q.argtypes = [P(Problem), ctypes.c_int, ctypes.c_int, ctypes.c_uint64, ctypes.c_uint32]
        _lib.orc_q.restype = ctypes.c_uint64
        _lib.orc_energy.argtypes = [P(Problem), ctypes.c_void_p, P(ctypes.c_uint64), P(ctypes.c_double)]
        _lib.orc_delta_replace.argtypes = [P(Problem), ctypes.c_void_p, ctypes.c_uint32, ctypes.c_uint32,
                                           ctypes.c_uint32, P(ctypes.c_uint64)]
        _lib.orc_optimize.argtypes = [P(Problem), ctypes.c_void_p, ctypes.c_void_p, P(Opt), ctypes.c_void_p,
                                      ctypes.c_void_p]
        _lib.orc_optimize.restype = ctypes.c_int
        _lib.orc_active_pixel.argtypes = [ctypes.c_uint32, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint32,
                                          ctypes.c_uint32]
        _lib.orc_active_pixel.restype = ctypes.c_uint32
        _lib.orc_gauss_kernel.argtypes = [ctypes.c_double, ctypes.c_void_p, ctypes.c_int]
        _lib.orc_gauss_kernel.restype = ctypes.c_int
        _lib.orc_denoised_rmse.argtypes = [P(Problem), ctypes.c_void_p, ctypes.c_uint32, ctypes.c_void_p,
                                           ctypes.c_uint32, ctypes.c_void_p]
        _lib.orc_denoised_rmse.restype = ctypes.c_int
        _lib.orc_error_spectrum.argtypes = [P(Problem), ctypes.c_void_p, ctypes.c_uint32, ctypes.c_void_p,
                                            ctypes.c_void_p]
        _lib.orc_error_spectrum.restype = ctypes.c_int
        _lib.orc_paper_key.argtypes = [ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint32]
        _lib.orc_paper_key.restype = ctypes.c_uint32
        _lib.orc_paper_couples.argtypes = [ctypes.c_void_p, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint32,
                                           ctypes.c_void_p]
        _lib.orc_paper_couples.restype = ctypes.c_int
        _lib.orc_paper_optimize.argtypes = [P(Problem), ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                            ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint64,
                                            ctypes.c_void_p, ctypes.c_void_p]
        _lib.orc_paper_optimize.restype = ctypes.c_int
        _lib.orc_bump_integral.argtypes = [ctypes.c_double] * 4
        _lib.orc_bump_integral.restype = ctypes.c_double
        _lib.orc_smooth_errors.argtypes = [P(Problem), ctypes.c_void_p, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_void_p,
                                           ctypes.c_void_p]
        _lib.orc_smooth_errors.restype = ctypes.c_int
        _lib.orc_denoised_rmse_images.argtypes = [ctypes.c_uint32, ctypes.c_uint32, ctypes.c_void_p, ctypes.c_void_p,
                                                  ctypes.c_uint32, ctypes.c_void_p]
        _lib.orc_denoised_rmse_images.restype = ctypes.c_int
        _lib.orc_error_spectrum_images.argtypes = [ctypes.c_uint32, ctypes.c_uint32, ctypes.c_void_p, ctypes.c_void_p,
                                                   ctypes.c_void_p]
        _lib.orc_error_spectrum_images.restype = ctypes.c_int
    return _lib


def _u128(lo: int, hi: int) -> int:
    return int(lo) | (int(hi) << 64)


def _i128(lo: int, hi: int) -> int:
    v = _u128(lo, hi)
    return v - (1 << 128) if v >> 127 else v


# ------------------------------------------------------------------------------------------
def philox4x32_10(ctr, key) -> tuple:
    """Philox4x32-10 (Salmon et al. 2011) -- counter-based RNG the north star names."""
    c = (ctypes.c_uint32 * 4)(*[int(v) & 0xFFFFFFFF for v in ctr])
    k = (ctypes.c_uint32 * 2)(*[int(v) & 0xFFFFFFFF for v in key])
    o = (ctypes.c_uint32 * 4)()
    lib().orc_philox4x32_10(c, k, o)
    return tuple(o)


def vdc_bits(k: int) -> int:
    """Van der Corput Phi(k) as a 32-bit numerator (§3.2 l.261-262)."""
    return lib().orc_vdc_bits(k)


def lattice(d1: int, d2: int, n: int) -> np.ndarray:
    """s^k = mod(Phi(k) d, 1), k < n, as uint32 fixed point [n, 2]."""
    out = np.zeros((n, 2), dtype=np.uint32)
    lib().orc_lattice(d1, d2, n, out.ctypes.data)
    return out


def sample(d1: int, d2: int, ux: int, uy: int, k: int) -> tuple:
    """Scrambled sample s^k_p = mod(s^k + u_p, 1) in fixed point (teaser PAPER.md l.54)."""
    o = (ctypes.c_uint32 * 2)()
    lib().orc_sample(d1, d2, ux, uy, k, o)
    return int(o[0]), int(o[1])


def paper_key(seed: int, t: int, P: int) -> int:
    """Per-pass XOR scramble key = Philox(seed; t,0,0,5)[0] & (P-1) (R25)."""
    return lib().orc_paper_key(seed, t, P)


def paper_couples(perm, key: int, budget: int) -> np.ndarray:
    """Couples of one pass, [budget/2, 2]: (perm[2c]^key, perm[2c+1]^key)."""
    perm = np.ascontiguousarray(perm, dtype=np.uint32)
    out = np.zeros(budget, np.uint32)
    if lib().orc_paper_couples(perm.ctypes.data, len(perm), key, budget, out.ctypes.data) != 0:
        raise ValueError("oracle rejected the couple arguments")
    return out.reshape(-1, 2)


def gauss_kernel(sigma: float) -> np.ndarray:
    """Normalised Gaussian kernel, radius ceil(4 sigma) (SPEC gaussian_kernel)."""
    r = int(np.ceil(4 * sigma))
    k = np.zeros((2 * r + 1) ** 2, np.float64)
    if lib().orc_gauss_kernel(sigma, k.ctypes.data, k.size) < 0:
        raise ValueError("bad sigma")
    return k.reshape(2 * r + 1, 2 * r + 1)


def iref(a: int, b: int, px: int, py: int) -> float:
    """Exact half-plane area inside [0,1]^2 (teaser 'I_ref')."""
    return lib().orc_iref(a, b, px, py)


def bump_integral(cx: float, cy: float, sx: float, sy: float) -> float:
    """Exact integral over [0,1]^2 of the Gaussian bump (separable erf product)."""
    return lib().orc_bump_integral(cx, cy, sx, sy)


def denoised_rmse_images(e: np.ndarray, sigmas) -> np.ndarray:
    """Evaluation criterion (§3.3) on error images e[ni][L][L] (plain convolution)."""
    e = np.ascontiguousarray(e, dtype=np.float64)
    ni, L = e.shape[0], e.shape[-1]
    sg = np.ascontiguousarray(sigmas, dtype=np.float64)
    out = np.zeros(len(sg), np.float64)
    if lib().orc_denoised_rmse_images(L, ni, e.ctypes.data, sg.ctypes.data, len(sg), out.ctypes.data):
        raise ValueError("bad arguments")
    return out


def error_spectrum_images(e: np.ndarray):
    """(S [L, L] mean power spectrum of the mean-subtracted images, radial profile [L/2])."""
    e = np.ascontiguousarray(e, dtype=np.float64)
    ni, L = e.shape[0], e.shape[-1]
    S = np.zeros((L, L), np.float64)
    prof = np.zeros(L // 2, np.float64)
    if lib().orc_error_spectrum_images(L, ni, e.ctypes.data, S.ctypes.data, prof.ctypes.data):
        raise ValueError("bad arguments")
    return S, prof


@dataclass
class OracleProblem:
    """One tile problem: bank + lattice + energy parameters (readings R2-R9)."""

    L: int
    T: int
    levels: tuple
    d1: int
    d2: int
    a: np.ndarray
    b: np.ndarray
    px: np.ndarray
    py: np.ndarray
    sigma_i: float = 2.1
    sigma_s: float = 1.0
    radius: int = 7
    form: int = 0          # 0 GF (north star), 1 Eq. 1 minimised, 2 Eq. 1 maximised

    def __post_init__(self):
        self.a = np.ascontiguousarray(self.a, dtype=np.int32)
        self.b = np.ascontiguousarray(self.b, dtype=np.int32)
        self.px = np.ascontiguousarray(self.px, dtype=np.uint32)
        self.py = np.ascontiguousarray(self.py, dtype=np.uint32)
        lv = (ctypes.c_uint32 * 8)(*(list(self.levels) + [0] * (8 - len(self.levels))))
        self._s = Problem(self.L, self.T, len(self.levels), lv, self.d1, self.d2,
                          self.a.ctypes.data, self.b.ctypes.data, self.px.ctypes.data, self.py.ctypes.data,
                          self.sigma_i, self.sigma_s, self.radius, self.form)

    @property
    def P(self) -> int:
        return self.L * self.L

    def ref(self):
        return ctypes.byref(self._s)

    # -- error vectors ---------------------------------------------------------------------
    def count1(self, ux: int, uy: int, i: int, N: int) -> int:
        return lib().orc_count1(self.ref(), ux, uy, i, N)

    def counts(self, U: np.ndarray) -> np.ndarray:
        """c[l][p][i] = #{k < N_l : f_i(mod(s^k + u_p, 1)) = 1}."""
        U = np.ascontiguousarray(U, dtype=np.uint32).reshape(-1, 2)
        P = U.shape[0]
        out = np.zeros((len(self.levels), P, self.T), dtype=np.uint8)
        lib().orc_counts(self.ref(), U.ctypes.data, P, out.ctypes.data)
        return out

    def references(self) -> np.ndarray:
        return np.array([iref(int(self.a[i]), int(self.b[i]), int(self.px[i]), int(self.py[i]))
                         for i in range(self.T)], dtype=np.float64)

    # -- energy ----------------------------------------------------------------------------
    def q(self, ox: int, oy: int, D: int, N: int) -> int:
        return lib().orc_q(self.ref(), ox, oy, D, N)

    def energy(self, c: np.ndarray):
        """(E_fixed as int, E_plain float) over counts c[l][p][i]."""
        c = np.ascontiguousarray(c, dtype=np.uint8)
        ef = (ctypes.c_uint64 * 2)()
        ep = ctypes.c_double()
        lib().orc_energy(self.ref(), c.ctypes.data, ef, ctypes.byref(ep))
        return _u128(ef[0], ef[1]), ep.value

    def delta_replace(self, c: np.ndarray, p: int, ux: int, uy: int) -> int:
        c = np.ascontiguousarray(c, dtype=np.uint8)
        d = (ctypes.c_uint64 * 2)()
        lib().orc_delta_replace(self.ref(), c.ctypes.data, p, ux, uy, d)
        return _i128(d[0], d[1])

    # -- evaluation criterion (§3.3) ------------------------------------------------
    def denoised_rmse(self, c: np.ndarray, level: int, sigmas) -> np.ndarray:
        """RMSE of the Gaussian-denoised test-integrand tiles, averaged over integrands (teaser (c))."""
        c = np.ascontiguousarray(c, dtype=np.uint8)
        sg = np.ascontiguousarray(sigmas, dtype=np.float64)
        out = np.zeros(len(sg), np.float64)
        if lib().orc_denoised_rmse(self.ref(), c.ctypes.data, level, sg.ctypes.data, len(sg), out.ctypes.data):
            raise ValueError("bad arguments")
        return out

    def smooth_errors(self, U: np.ndarray, level: int, bumps) -> np.ndarray:
        """Errors e_i(p) [nb][L][L] of the Gaussian-bump integrands (cx, cy, sx, sy) at progressive
        level `level` of the tile U: 1/N sum_k f_i(s^k_p) - I_i (§3.5 l.309-313)."""
        U = np.ascontiguousarray(U, dtype=np.uint32).reshape(-1, 2)
        bm = np.ascontiguousarray(bumps, dtype=np.float64).reshape(-1, 4)
        out = np.zeros((len(bm), self.L, self.L), np.float64)
        if lib().orc_smooth_errors(self.ref(), U.ctypes.data, level, len(bm), bm.ctypes.data, out.ctypes.data):
            raise ValueError("bad arguments")
        return out

    def error_spectrum(self, c: np.ndarray, level: int):
        """(S [L, L] mean power spectrum of the mean-subtracted error, radial profile [L/2])."""
        c = np.ascontiguousarray(c, dtype=np.uint8)
        S = np.zeros((self.L, self.L), np.float64)
        prof = np.zeros(self.L // 2, np.float64)
        if lib().orc_error_spectrum(self.ref(), c.ctypes.data, level, S.ctypes.data, prof.ctypes.data):
            raise ValueError("bad arguments")
        return S, prof

    # -- optimisation ----------------------------------------------------------------------
    def optimize(self, U: np.ndarray, c: np.ndarray | None = None, *, mode: int = 0, passes: int = 1,
                 first_pass: int = 0, K: int = 1, seed: int = 3, max_steps: int = 0,
                 gauss_seidel: bool = False, energy_each_pass: bool = True, log: bool = False):
        """Run the greedy independent-set optimiser.  Returns (U, c, stats list, accept log)."""
        U = np.array(U, dtype=np.uint32).reshape(-1, 2).copy()
        c = self.counts(U) if c is None else np.array(c, dtype=np.uint8, copy=True)
        M = (self.L // 8) ** 2
        st = (Stats * max(passes, 1))()
        acc = np.zeros((passes, 64, M), dtype=np.uint8) if log else None
        o = Opt(mode, passes, first_pass, K, seed, max_steps, int(gauss_seidel), int(energy_each_pass))
        rc = lib().orc_optimize(self.ref(), U.ctypes.data, c.ctypes.data, ctypes.byref(o), st,
                                acc.ctypes.data if acc is not None else None)
        if rc != 0:
            raise ValueError("oracle rejected the optimisation arguments")
        stats = [dict(accepted=s.accepted, proposed=s.proposed, E_plain=s.E_plain,
                      E_fixed=_u128(s.E_fixed[0], s.E_fixed[1]), dE_sum=_i128(s.dE_sum[0], s.dE_sum[1]))
                 for s in list(st)[:passes]]
        return U, c, stats, acc

    def paper_optimize(self, U: np.ndarray, perm, *, budget: int | None = None, passes: int = 1,
                       first_pass: int = 0, seed: int = 3, c: np.ndarray | None = None, log: bool = False,
                       energy_each_pass: bool = True):
        """Paper-verbatim parallel swaps against the pass-start snapshot (§3.4 l.291-307).
        Returns (U, c, stats list, accept log [passes, budget/2] or None)."""
        U = np.array(U, dtype=np.uint32).reshape(-1, 2).copy()
        c = self.counts(U) if c is None else np.array(c, dtype=np.uint8, copy=True)
        perm = np.ascontiguousarray(perm, dtype=np.uint32)
        budget = self.P // 4 if budget is None else budget
        st = (Stats * max(passes, 1))()
        acc = np.zeros((passes, max(budget // 2, 1)), dtype=np.uint8) if log else None
        rc = lib().orc_paper_optimize(self.ref(), U.ctypes.data, c.ctypes.data, perm.ctypes.data, budget, passes,
                                      first_pass, seed, st if energy_each_pass else None,
                                      acc.ctypes.data if acc is not None else None)
        if rc != 0:
            raise ValueError("oracle rejected the paper-mode arguments")
        stats = [dict(accepted=s.accepted, proposed=s.proposed, E_plain=s.E_plain,
                      E_fixed=_u128(s.E_fixed[0], s.E_fixed[1]), dE_sum=_i128(s.dE_sum[0], s.dE_sum[1]))
                 for s in list(st)[:passes]]
        return U, c, stats, acc

    def active_pixel(self, seed: int, t: int, s: int, m: int) -> int:
        return lib().orc_active_pixel(self.L, seed, t, s, m)
