"""Thin ctypes binding of the C-ABI in ``include/bn.h`` (argument marshalling only).

Every step of the hot path runs in the CUDA kernels of ``libbn.so``; this module never
computes anything of the method and has no fallback: if the library is missing or no CUDA
device is present, calls raise.  Names mirror the C entry points (``bn_set_lattice`` ->
``Sampler.set_lattice``...).  Arrays may be numpy (host) or torch CUDA tensors (device,
passed by ``data_ptr()``); the stream is torch's current stream unless given.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("BN_LIB") or os.path.join(_HERE, "libbn.so")  # BN_LIB: an experiment build

BN_OK, BN_EINVAL, BN_ECUDA, BN_ENCCL, BN_ENOMEM, BN_ESTATE = range(6)
REDRAW, SWAP, PAPER_SWAP = 0, 1, 2
E_GF, E_EQ1, E_EQ1_MAX = 0, 1, 2
_STATUS = {1: "EINVAL", 2: "ECUDA", 3: "ENCCL", 4: "ENOMEM", 5: "ESTATE"}

#: every entry point declared in include/bn.h (checked by tests/test_abi.py)
SYMBOLS = ("bn_create", "bn_destroy", "bn_last_error", "bn_version", "bn_set_lattice", "bn_set_bank",
           "bn_get_references", "bn_set_energy", "bn_set_tile", "bn_get_tile", "bn_eval_counts", "bn_energy",
           "bn_optimize", "bn_comm_init", "bn_comm_unique_id", "bn_launch_count", "bn_profile_enable",
           "bn_profile_get", "bn_window_distances", "bn_set_permutation",
           "bn_set_energy_form", "bn_eval_quality", "bn_check", "bn_eval_smooth")
KERNELS = ("counts", "gather", "gram", "lut", "decide", "stats", "commit", "tail")


class BNError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"bn {_STATUS.get(code, code)}: {msg}")
        self.code = code


class OptParams(ctypes.Structure):
    _fields_ = [("mode", ctypes.c_uint32), ("passes", ctypes.c_uint32), ("first_pass", ctypes.c_uint32),
                ("K", ctypes.c_uint32), ("seed", ctypes.c_uint64), ("budget", ctypes.c_uint32),
                ("reserved", ctypes.c_uint32)]


class PassStats(ctypes.Structure):
    _fields_ = [("accepted", ctypes.c_uint32), ("proposed", ctypes.c_uint32), ("E", ctypes.c_double),
                ("E_fixed", ctypes.c_uint64 * 2), ("dE_sum", ctypes.c_uint64 * 2)]


_lib = None


def load_library(path: str = LIB_PATH):
    """Load libbn.so; raises (never falls back) if it is missing."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(f"{path} is missing: run `python -m paper_2105_12620_b200.build` "
                          f"(or __graft_entry__.build()); there is no CPU fallback")
    lib = ctypes.CDLL(path)
    vp, u32, u64, i32 = ctypes.c_void_p, ctypes.c_uint32, ctypes.c_uint64, ctypes.c_int32
    sig = {
        "bn_create": ([ctypes.POINTER(vp), ctypes.c_int, ctypes.c_size_t], ctypes.c_int),
        "bn_destroy": ([vp], None),
        "bn_last_error": ([vp], ctypes.c_char_p),
        "bn_version": ([], ctypes.c_char_p),
        "bn_set_lattice": ([vp, u32, u32, vp, u32], ctypes.c_int),
        "bn_set_bank": ([vp, u32, vp, vp, vp, vp, u32, u32], ctypes.c_int),
        "bn_get_references": ([vp, vp], ctypes.c_int),
        "bn_set_energy": ([vp, ctypes.c_double, ctypes.c_double, i32], ctypes.c_int),
        "bn_set_tile": ([vp, u32, vp, ctypes.c_int], ctypes.c_int),
        "bn_get_tile": ([vp, vp, ctypes.c_int], ctypes.c_int),
        "bn_eval_counts": ([vp, vp, ctypes.c_int], ctypes.c_int),
        "bn_energy": ([vp, ctypes.POINTER(ctypes.c_double), vp], ctypes.c_int),
        "bn_optimize": ([vp, ctypes.POINTER(OptParams), vp, vp], ctypes.c_int),
        "bn_comm_init": ([vp, vp, ctypes.c_int, ctypes.c_int], ctypes.c_int),
        "bn_comm_unique_id": ([vp], ctypes.c_int),
        "bn_check": ([vp], ctypes.c_int),
        "bn_eval_smooth": ([vp, u32, u32, vp, vp, u32, vp, vp, vp, vp], ctypes.c_int),
        "bn_launch_count": ([vp], u64),
        "bn_profile_enable": ([vp, ctypes.c_int], ctypes.c_int),
        "bn_window_distances": ([vp, vp, ctypes.c_int], ctypes.c_int),
        "bn_set_permutation": ([vp, vp, u32], ctypes.c_int),
        "bn_set_energy_form": ([vp, u32], ctypes.c_int),
        "bn_eval_quality": ([vp, u32, vp, u32, vp, vp, vp], ctypes.c_int),
        "bn_profile_get": ([vp, u32, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(u64)], ctypes.c_int),
    }
    for name, (args, res) in sig.items():
        f = getattr(lib, name)
        f.argtypes = args
        f.restype = res
    _lib = lib
    return lib


def _ptr(x, n: int | None = None, dtype=None):
    """(pointer, is_device) of a numpy array or torch tensor (contiguous).  With `n` / `dtype`,
    the buffer must hold exactly n elements of that numpy dtype (the C side trusts the size)."""
    if isinstance(x, np.ndarray):
        if not x.flags["C_CONTIGUOUS"]:
            raise ValueError("array must be C-contiguous")
        got_dt, got_n, ptr, dev = x.dtype, x.size, x.ctypes.data, 0
    elif hasattr(x, "data_ptr"):
        if not x.is_contiguous():
            raise ValueError("tensor must be contiguous")
        got_dt = np.dtype(str(x.dtype).replace("torch.", ""))
        got_n, ptr, dev = x.numel(), x.data_ptr(), int(x.is_cuda)
    else:
        raise TypeError(f"unsupported buffer type {type(x)}")
    if dtype is not None and got_dt != np.dtype(dtype):
        raise TypeError(f"buffer dtype {got_dt}, expected {np.dtype(dtype)}")
    if n is not None and got_n != n:
        raise ValueError(f"buffer holds {got_n} elements, expected {n}")
    return ptr, dev


def comm_unique_id() -> bytes:
    lib = load_library()
    buf = ctypes.create_string_buffer(128)
    rc = lib.bn_comm_unique_id(buf)
    if rc:
        raise BNError(rc, "ncclGetUniqueId failed")
    return buf.raw


class Sampler:
    """One tile problem on one GPU (one ``bn_ctx``)."""

    def __init__(self, device: int = 0, stream: int | None = None):
        self._lib = load_library()
        if stream is None:
            import torch

            torch.cuda.set_device(device)
            stream = torch.cuda.current_stream(device).cuda_stream
        self._ctx = ctypes.c_void_p()
        rc = self._lib.bn_create(ctypes.byref(self._ctx), device, stream)
        if rc:
            raise BNError(rc, f"bn_create(device={device}) failed")
        self.device, self.stream = device, stream
        self.L = self.T = self.Ts = 0
        self.levels: tuple = ()
        self.radius = 7

    def close(self):
        if getattr(self, "_ctx", None) and self._ctx.value:
            self._lib.bn_destroy(self._ctx)
            self._ctx = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, rc: int):
        if rc:
            raise BNError(rc, self._lib.bn_last_error(self._ctx).decode())

    # ------------------------------------------------------------------------------ setup
    def set_lattice(self, d1: int, d2: int, spp_levels):
        lv = np.ascontiguousarray(spp_levels, dtype=np.uint32)
        self._check(self._lib.bn_set_lattice(self._ctx, d1, d2, lv.ctypes.data, len(lv)))
        self.levels = tuple(int(v) for v in lv)

    def set_bank(self, a, b, px, py, t_begin: int = 0, t_end: int | None = None):
        a, b = (np.ascontiguousarray(v, dtype=np.int32) for v in (a, b))
        px, py = (np.ascontiguousarray(v, dtype=np.uint32) for v in (px, py))
        T = len(a)
        t_end = T if t_end is None else t_end
        self._check(self._lib.bn_set_bank(self._ctx, T, a.ctypes.data, b.ctypes.data, px.ctypes.data,
                                          py.ctypes.data, t_begin, t_end))
        self.T, self.Ts = T, t_end - t_begin

    def get_references(self) -> np.ndarray:
        out = np.zeros(self.Ts, np.float64)
        self._check(self._lib.bn_get_references(self._ctx, out.ctypes.data))
        return out

    def set_energy(self, sigma_i: float = 2.1, sigma_s: float = 1.0, radius: int = 7):
        self._check(self._lib.bn_set_energy(self._ctx, sigma_i, sigma_s, radius))
        self.radius = radius

    def set_energy_form(self, form: int = E_GF):
        """Energy g(D): E_GF (default), E_EQ1 (Eq. 1 as written, minimised), E_EQ1_MAX (Eq. 1 maximised)."""
        self._check(self._lib.bn_set_energy_form(self._ctx, form))

    def set_tile(self, L: int, u_xy):
        ptr, dev = _ptr(u_xy, 2 * L * L, np.uint32)
        self._check(self._lib.bn_set_tile(self._ctx, L, ptr, dev))
        self.L = L

    def get_tile(self, out=None):
        if out is None:
            out = np.zeros((self.L * self.L, 2), np.uint32)
        ptr, dev = _ptr(out, 2 * self.L * self.L, np.uint32)
        self._check(self._lib.bn_get_tile(self._ctx, ptr, dev))
        return out

    def eval_counts(self, out=None):
        if out is None:
            out = np.zeros((len(self.levels), self.L * self.L, self.Ts), np.uint8)
        ptr, dev = _ptr(out, len(self.levels) * self.L * self.L * self.Ts, np.uint8)
        self._check(self._lib.bn_eval_counts(self._ctx, ptr, dev))
        return out

    def energy(self):
        """(E_fixed as Python int, E as float)."""
        E = ctypes.c_double()
        ef = (ctypes.c_uint64 * 2)()
        self._check(self._lib.bn_energy(self._ctx, ctypes.byref(E), ef))
        return int(ef[0]) | (int(ef[1]) << 64), E.value

    def set_permutation(self, perm):
        """Precomputed pixel permutation of the paper-verbatim mode."""
        perm = np.ascontiguousarray(perm, dtype=np.uint32)
        self._check(self._lib.bn_set_permutation(self._ctx, perm.ctypes.data, len(perm)))

    def optimize(self, passes: int, seed: int, mode: int = REDRAW, first_pass: int = 0, K: int = 1,
                 stats: bool = True, log: bool = False, budget: int = 0):
        """Run passes; returns (list of per-pass dicts or None, accept log or None).  The log is
        [passes, 64, M] for REDRAW/SWAP and [passes, budget/2] (couple flags) for PAPER_SWAP."""
        prm = OptParams(mode, passes, first_pass, K, seed, budget, 0)
        st = (PassStats * max(passes, 1))() if stats else None
        M = (self.L // 8) ** 2
        lg = np.zeros((passes, 64, M), np.uint8) if log else None
        self._check(self._lib.bn_optimize(self._ctx, ctypes.byref(prm), st,
                                          lg.ctypes.data if lg is not None else None))
        out = None
        if stats:
            out = []
            for s in list(st)[:passes]:
                d = int(s.dE_sum[0]) | (int(s.dE_sum[1]) << 64)
                out.append(dict(accepted=s.accepted, proposed=s.proposed, E=s.E,
                                E_fixed=int(s.E_fixed[0]) | (int(s.E_fixed[1]) << 64),
                                dE_sum=d - (1 << 128) if d >> 127 else d))
        if lg is not None and mode == PAPER_SWAP:
            ncp = (budget or self.L * self.L // 4) // 2
            lg = lg.reshape(passes, -1)[:, :ncp].copy()
        return out, lg

    def eval_quality(self, level: int = 0, sigmas=None, spectrum: bool = True):
        """Paper's evaluation criterion (§3.3): (denoised RMSE per sigma, mean error power
        spectrum [L, L] or None, radial profile [L/2] or None).  Default sigmas: 16 log-spaced in
        [0.25, 20]."""
        sg = np.geomspace(0.25, 20.0, 16) if sigmas is None else np.ascontiguousarray(sigmas, dtype=np.float64)
        sg = np.ascontiguousarray(sg, dtype=np.float64)
        r = np.zeros(len(sg), np.float64)
        S = np.zeros((self.L, self.L), np.float64) if spectrum else None
        prof = np.zeros(self.L // 2, np.float64) if spectrum else None
        self._check(self._lib.bn_eval_quality(self._ctx, level, sg.ctypes.data, len(sg), r.ctypes.data,
                                              S.ctypes.data if S is not None else None,
                                              prof.ctypes.data if prof is not None else None))
        return r, S, prof

    def eval_smooth(self, bumps, level: int = 0, sigmas=None, spectrum: bool = True):
        """Evaluation criterion for the smooth Gaussian-bump integrands (§3.5): (denoised RMSE
        per sigma, spectrum [L, L] or None, radial profile [L/2] or None, exact references [n]).
        bumps: [n][4] = (cx, cy, sx, sy); default sigmas: 16 log-spaced in [0.25, 20]."""
        bm = np.ascontiguousarray(bumps, dtype=np.float64).reshape(-1, 4)
        sg = np.geomspace(0.25, 20.0, 16) if sigmas is None else np.ascontiguousarray(sigmas, dtype=np.float64)
        sg = np.ascontiguousarray(sg, dtype=np.float64)
        r = np.zeros(len(sg), np.float64)
        S = np.zeros((self.L, self.L), np.float64) if spectrum else None
        prof = np.zeros(self.L // 2, np.float64) if spectrum else None
        ref = np.zeros(len(bm), np.float64)
        self._check(self._lib.bn_eval_smooth(self._ctx, level, len(bm), bm.ctypes.data, sg.ctypes.data, len(sg),
                                             r.ctypes.data, S.ctypes.data if S is not None else None,
                                             prof.ctypes.data if prof is not None else None, ref.ctypes.data))
        return r, S, prof, ref

    def window_distances(self, out=None):
        """Partial (this bank shard) window distances D_l(p, p+o), [levels, P, H] int32,
        H = 2R^2 + 2R for the radius of the last set_energy."""
        H = 2 * self.radius * self.radius + 2 * self.radius
        n = len(self.levels) * self.L * self.L * H
        if out is None:
            out = np.zeros((len(self.levels), self.L * self.L, H), np.int32)
        ptr, dev = _ptr(out, n, np.int32)
        self._check(self._lib.bn_window_distances(self._ctx, ptr, dev))
        return out

    def check(self):
        """Synchronise and raise BNError(BN_ESTATE) if any device invariant failed since the last read."""
        self._check(self._lib.bn_check(self._ctx))

    def comm_init(self, uid: bytes, rank: int, world: int):
        self._check(self._lib.bn_comm_init(self._ctx, uid, rank, world))

    def launch_count(self) -> int:
        return int(self._lib.bn_launch_count(self._ctx))

    def profile_enable(self, on: bool = True):
        self._check(self._lib.bn_profile_enable(self._ctx, int(on)))

    def profile(self) -> dict:
        """{kernel: (total_ms, launches)} accumulated since profile_enable(True)."""
        out = {}
        for i, name in enumerate(KERNELS):
            ms, n = ctypes.c_double(), ctypes.c_uint64()
            self._check(self._lib.bn_profile_get(self._ctx, i, ctypes.byref(ms), ctypes.byref(n)))
            out[name] = (ms.value, int(n.value))
        return out


def version() -> str:
    return load_library().bn_version().decode()
