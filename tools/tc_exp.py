"""Time the window-Gram kernel alone (bn_window_distances) under the current BN_* environment."""
import sys, time
sys.path.insert(0, '.')
import torch
import synth
from paper_2105_12620_b200 import bn
cfg = synth.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C3"]
U, (a, b, px, py) = synth.problem_inputs(cfg)
s = bn.Sampler(0)
s.set_lattice(synth.D1, synth.D2, cfg.levels); s.set_bank(a, b, px, py); s.set_energy(2.1, 1.0, 7); s.set_tile(cfg.L, U)
out = torch.empty((len(cfg.levels), cfg.L * cfg.L, 112), dtype=torch.int32, device="cuda")
for _ in range(3): s.window_distances(out=out)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); n = 20
for _ in range(n): s.window_distances(out=out)
e1.record(); torch.cuda.synchronize()
print(f"window_distances (gram + export): {e0.elapsed_time(e1)/n:.4f} ms")
