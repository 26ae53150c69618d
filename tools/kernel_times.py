"""Per-kernel device times of N passes on one config (profiling events), no checks: also usable
with timing-probe builds (BN_LIB=...) whose results are wrong by construction.
usage: python tools/kernel_times.py [C3] [swap|redraw] [passes]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
from paper_2105_12620_b200 import bn  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C3"
mode = {"swap": 1, "redraw": 0}[sys.argv[2]] if len(sys.argv) > 2 else synth.CONFIGS[name].mode
passes = int(sys.argv[3]) if len(sys.argv) > 3 else 10
cfg = synth.CONFIGS[name]
U, (a, b, px, py) = synth.problem_inputs(cfg)
s = bn.Sampler(0)
s.set_lattice(synth.D1, synth.D2, cfg.levels)
s.set_bank(a, b, px, py)
s.set_energy(2.1, 1.0, 7)
s.set_tile(cfg.L, U)
s.optimize(3, 3, mode=mode, stats=False)
s.profile_enable(True)
s.optimize(passes, 3, mode=mode, first_pass=3, stats=False)
prof = s.profile()
print(os.environ.get("BN_LIB", "libbn.so").split("/")[-1], os.environ.get("BN_NARROW", ""),
      {k: round(v[0] / passes * 1e3, 1) for k, v in prof.items() if v[1]})
