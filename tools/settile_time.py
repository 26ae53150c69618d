"""Device time of bn_set_tile (counts rebuild, + the narrow pack) per call, no checks (timing probes).
usage: python tools/settile_time.py [C3] [reps]"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2105_12620_b200 import bn  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C3"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
cfg = synth.CONFIGS[name]
U, (a, b, px, py) = synth.problem_inputs(cfg)
s = bn.Sampler(0)
s.set_lattice(synth.D1, synth.D2, cfg.levels)
s.set_bank(a, b, px, py)
s.set_energy(2.1, 1.0, 7)
for _ in range(3):
    s.set_tile(cfg.L, U)
    s.energy()
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(reps):
    s.set_tile(cfg.L, U)
    s.energy()  # resolves the narrow speculation (first consumer)
torch.cuda.synchronize()
t1 = time.perf_counter()
s.close()
print(os.environ.get("BN_LIB", "libbn.so").split("/")[-1], name, os.environ.get("BN_NARROW", ""),
      f"{(t1 - t0) / reps * 1e3:.3f} ms per set_tile + energy")
