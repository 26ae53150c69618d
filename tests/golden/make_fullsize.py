"""Write the full-BASELINE-size oracle goldens `tests/golden/fullsize_*.json`.

TEST INFRASTRUCTURE.  Calls only `oracle/` (and the seeded input generators in `synth/`), never the
CUDA path: every stored value is the CPU oracle's.  Run on CPU (one process per job):

    python tests/golden/make_fullsize.py [job ...]

Per job (config, pair, mode, passes; SURVEY.md §8(d) parity plan: C2 20 passes, C3 2 SWAP passes +
2 REDRAW passes, C4 1 pass x 8 pairs, C5 1 pass) the file holds the oracle's
  * sha256 of the initial counts [level][P][T] (the error vectors of the input tile),
  * per pass: accepted, proposed, exact E_fixed and dE_sum (decimal), E_plain, sha256 of the tile
    U [P][2] after the pass and the complete accept log [64][M] (np.packbits, base64),
  * sha256 of the final counts.
The GPU tests (`tests/test_gpu_fullsize.py`) run the same passes through the C-ABI and compare.
"""
from __future__ import annotations

import base64
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

# name -> (config, pair, mode, passes)
JOBS = {
    "C2_swap": ("C2", 0, 1, 20),
    "C3_swap": ("C3", 0, 1, 2),
    "C3_redraw": ("C3", 0, 0, 2),
    **{f"C4_pair{j}_swap": ("C4", j, 1, 1) for j in range(8)},
    "C5_swap": ("C5", 0, 1, 1),
}


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def path(name: str) -> str:
    return os.path.join(HERE, f"fullsize_{name}.json")


def run(name: str) -> str:
    from oracle import oracle

    cfg_name, pair, mode, passes = JOBS[name]
    cfg = synth.CONFIGS[cfg_name]
    U, (a, b, px, py) = synth.problem_inputs(cfg, pair)
    seed = synth.opt_seed(cfg, pair)
    o = oracle.OracleProblem(cfg.L, cfg.T, tuple(cfg.levels), synth.D1, synth.D2, a, b, px, py)
    t0 = time.time()
    c = o.counts(U)
    out = dict(job=name, config=cfg_name, pair=pair, mode=mode, passes=passes, seed=seed, L=cfg.L, T=cfg.T,
               levels=list(cfg.levels), counts0_sha256=sha(c), per_pass=[])
    # one oracle call per pass (resumed with first_pass) so every pass's tile can be hashed
    for t in range(passes):
        U, c, st, lg = o.optimize(U, c, mode=mode, passes=1, first_pass=t, seed=seed, log=True)
        s = st[0]
        out["per_pass"].append(dict(
            accepted=s["accepted"], proposed=s["proposed"], E_fixed=str(s["E_fixed"]), dE_sum=str(s["dE_sum"]),
            E_plain=s["E_plain"], U_sha256=sha(U),
            log_packbits_b64=base64.b64encode(np.packbits(lg[0].reshape(-1))).decode()))
    out["counts_final_sha256"] = sha(c)
    out["oracle_seconds"] = round(time.time() - t0, 1)
    with open(path(name), "w") as f:
        json.dump(out, f, indent=1)
    return f"{name}: {out['oracle_seconds']} s"


def load(name: str) -> dict:
    with open(path(name)) as f:
        return json.load(f)


def unpack_log(b64: str, M: int) -> np.ndarray:
    bits = np.unpackbits(np.frombuffer(base64.b64decode(b64), np.uint8))
    return bits[:64 * M].reshape(64, M)


if __name__ == "__main__":
    names = sys.argv[1:] or list(JOBS)
    # longest first
    names.sort(key=lambda n: {"C5": 0, "C3": 1}.get(JOBS[n][0], 2))
    with Pool(min(len(names), os.cpu_count() or 1)) as pool:
        for r in pool.imap_unordered(run, names):
            print(r, flush=True)
