"""Time k_counts alone (bn_eval_counts path: set_tile recount) under the current BN_* environment."""
import sys
sys.path.insert(0, '.')
import torch
import synth
from paper_2105_12620_b200 import bn
cfg = synth.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C3"]
U, (a, b, px, py) = synth.problem_inputs(cfg)
s = bn.Sampler(0)
s.set_lattice(synth.D1, synth.D2, cfg.levels); s.set_bank(a, b, px, py); s.set_energy(2.1, 1.0, 7)
s.profile_enable(True)
for _ in range(3):
    s.set_tile(cfg.L, U); s.eval_counts()
torch.cuda.synchronize()
s.profile_enable(True)
n = 10
for _ in range(n):
    s.set_tile(cfg.L, U); s.eval_counts()
torch.cuda.synchronize()
prof = s.profile()
print({k: round(v[0] / v[1], 4) for k, v in prof.items() if v[1]})
