"""Paper's evaluation criterion on GPU-optimised tiles (§3.3, teaser Fig. 1(c) analogue).

For one tile problem it runs, on the GPU, the random initial tile ("random scrambling", the white-
noise baseline of Fig. 1(c)) and the tiles left by P passes of each optimiser mode (greedy SWAP,
paper-verbatim snapshot couples, greedy REDRAW), and reports the denoised-RMSE curve (16
log-spaced sigmas in [0.25, 20]) and the radial error power profile of each, plus the time of the
bn_eval_quality call.  With --smooth N it also evaluates every tile on N smooth Gaussian-bump
integrands (§3.5 "even for low frequency integrands"; bn_eval_smooth), which no optimiser
sees.  The paper prints no numbers for this figure (parity unpinned); the output is the
qualitative ordering.

    python tools/eval_curve.py [--L 64] [--T 256] [--spp 16] [--passes 40] [--out profiles/...json]
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import synth  # noqa: E402
from paper_2105_12620_b200 import bn  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--L", type=int, default=64)
    ap.add_argument("--T", type=int, default=256)
    ap.add_argument("--spp", type=int, default=16)
    ap.add_argument("--passes", type=int, default=40)
    ap.add_argument("--smooth", type=int, default=0, help="smooth Gaussian-bump evaluation integrands")
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "eval_curve.json"))
    args = ap.parse_args()
    import torch

    L, T = args.L, args.T
    a, b, px, py = synth.make_bank(T, 2)
    U0 = synth.make_tile(L, 1)
    sig = np.geomspace(0.25, 20.0, 16)
    res = {"config": {"L": L, "T": T, "spp": args.spp, "passes": args.passes, "sigmas": sig.tolist(),
                      "bank_seed": 2, "tile_seed": 1, "opt_seed": 3}, "curves": {}}
    for name, mode, passes in (("random", None, 0), ("swap", bn.SWAP, args.passes),
                               ("paper", bn.PAPER_SWAP, 4 * args.passes), ("redraw", bn.REDRAW, args.passes)):
        s = bn.Sampler(0)
        s.set_lattice(synth.D1, synth.D2, [args.spp])
        s.set_bank(a, b, px, py)
        s.set_energy(2.1, 1.0, 7)
        s.set_tile(L, U0)
        if mode == bn.PAPER_SWAP:
            s.set_permutation(synth.make_permutation(L * L, 3))
        E0 = s.energy()[1]
        if mode is not None:
            s.optimize(passes, 3, mode=mode, stats=False)
        torch.cuda.synchronize()
        r, S, prof = s.eval_quality(0, sig)  # first call allocates the work buffers
        t0 = time.perf_counter()
        r, S, prof = s.eval_quality(0, sig)
        dt = time.perf_counter() - t0
        res["curves"][name] = {"passes": passes, "E_before": E0, "E_after": s.energy()[1], "rmse": r.tolist(),
                               "radial_profile": prof.tolist(), "eval_ms": 1e3 * dt}
        if args.smooth:
            rs, _, ps, _ = s.eval_smooth(synth.make_bumps(args.smooth, 5), 0, sig)
            res["curves"][name]["smooth"] = {"n_bumps": args.smooth, "bump_seed": 5, "rmse": rs.tolist(),
                                             "radial_profile": ps.tolist()}
            print(f"        smooth: rmse(1, 2, 5) = " + ", ".join(f"{rs[np.argmin(abs(sig - v))]:.3e}" for v in (1, 2, 5))
                  + f"   low/mid power {np.mean(ps[:L // 16]) / np.mean(ps[L // 4:3 * L // 8]):.3f}", flush=True)
        s.close()
        print(f"{name:7s} passes {passes:4d}  E {E0:.1f} -> {res['curves'][name]['E_after']:.1f}  "
              f"rmse(0.25, 1, 2, 5, 20) = " + ", ".join(f"{r[np.argmin(abs(sig - v))]:.3e}" for v in (0.25, 1, 2, 5, 20))
              + f"   low/mid power {np.mean(prof[:L // 16]) / np.mean(prof[L // 4:3 * L // 8]):.3f}"
              + f"   eval {1e3 * dt:.1f} ms", flush=True)
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    with open(args.out, "w") as f:
        json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
