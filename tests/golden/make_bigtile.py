"""Oracle goldens for the largest tiles the API accepts (L = 1024 and 2048; T = 8 ragged-free, one
4-spp level): one REDRAW and one SWAP pass each, from `tests/golden/bigtile_*.json`.

TEST INFRASTRUCTURE.  Calls only `oracle/` and the seeded generators in `synth/` (never the CUDA
path).  The accept logs (64 x L^2/64 bits) are stored as sha256 digests, like the tiles and counts.
Run on CPU:  python tests/golden/make_bigtile.py [L ...]   (~45 s per pass at L = 1024, ~160 s at 2048)
"""
from __future__ import annotations

import hashlib
import json
import os
import sys
import time
from multiprocessing import Pool

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import synth  # noqa: E402

T, LEVELS, BANK_SEED, TILE_SEED, OPT_SEED = 8, (4,), 2, 1, 5
JOBS = {f"L{L}_{m}": (L, mode) for L in (1024, 2048) for m, mode in (("redraw", 0), ("swap", 1))}


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def path(name: str) -> str:
    return os.path.join(HERE, f"bigtile_{name}.json")


def inputs(L: int):
    return synth.make_tile(L, TILE_SEED), synth.make_bank(T, BANK_SEED)


def run(name: str) -> str:
    from oracle import oracle

    L, mode = JOBS[name]
    U, (a, b, px, py) = inputs(L)
    o = oracle.OracleProblem(L, T, LEVELS, synth.D1, synth.D2, a, b, px, py)
    t0 = time.time()
    c = o.counts(U)
    U1, c1, st, lg = o.optimize(U, c, mode=mode, passes=1, seed=OPT_SEED, log=True)
    s = st[0]
    out = dict(job=name, L=L, T=T, levels=list(LEVELS), mode=mode, seed=OPT_SEED, counts0_sha256=sha(c),
               accepted=s["accepted"], proposed=s["proposed"], E_fixed=str(s["E_fixed"]), dE_sum=str(s["dE_sum"]),
               E_plain=s["E_plain"], U_sha256=sha(U1), log_sha256=sha(np.asarray(lg[0], np.uint8)),
               counts_final_sha256=sha(c1), oracle_seconds=round(time.time() - t0, 1))
    with open(path(name), "w") as f:
        json.dump(out, f, indent=1)
    return f"{name}: {out['oracle_seconds']} s"


def load(name: str) -> dict:
    with open(path(name)) as f:
        return json.load(f)


if __name__ == "__main__":
    Ls = [int(x) for x in sys.argv[1:]] or [1024, 2048]
    names = [n for n in JOBS if JOBS[n][0] in Ls]
    with Pool(len(names)) as pool:
        for r in pool.imap_unordered(run, names):
            print(r, flush=True)
