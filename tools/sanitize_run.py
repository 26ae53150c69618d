"""Small runs of every default kernel for compute-sanitizer (memcheck / racecheck / synccheck):
set_tile counts, SWAP passes (gather, window Gram, energy terms, fused tail or cluster decide +
commit-gather), REDRAW passes (prefetched counts, cluster decide, commit), the paper mode, an
L = 256 tile (bit-flag cluster decide), narrow rows, best-of-K and the evaluation criterion.
usage: compute-sanitizer --tool memcheck python tools/sanitize_run.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
from paper_2105_12620_b200 import bn  # noqa: E402


def ctx(L, T, levels, seed=1):
    a, b, px, py = synth.make_bank(T, seed + 1)
    s = bn.Sampler(0)
    s.set_lattice(synth.D1, synth.D2, levels)
    s.set_bank(a, b, px, py)
    s.set_energy(2.1, 1.0, 7)
    s.set_tile(L, synth.make_tile(L, seed))
    return s


runs = []
s = ctx(32, 100, (4, 16))
runs.append(("swap", s.optimize(3, 5, mode=bn.SWAP)[0][-1]["E_fixed"]))
runs.append(("redraw", s.optimize(3, 6, mode=bn.REDRAW, first_pass=3)[0][-1]["E_fixed"]))
s.set_permutation(synth.make_permutation(32 * 32, 7))
runs.append(("paper", s.optimize(2, 7, mode=bn.PAPER_SWAP, first_pass=6)[0][-1]["E_fixed"]))
runs.append(("best_of_3", s.optimize(1, 8, mode=bn.REDRAW, K=3, first_pass=8)[0][-1]["E_fixed"]))
runs.append(("quality", float(s.eval_quality(0, [1.0, 4.0], spectrum=True)[0][0])))
s.close()
s = ctx(256, 64, (16,), seed=3)  # L = 256: the bit-flag cluster decisions
runs.append(("swap_L256", s.optimize(2, 9, mode=bn.SWAP)[0][-1]["E_fixed"]))
runs.append(("redraw_L256", s.optimize(1, 10, mode=bn.REDRAW, first_pass=2)[0][-1]["E_fixed"]))
s.close()
os.environ["BN_NARROW"] = "1"  # narrow rows (e2m1 / e3m2) through the same path
s = ctx(32, 130, (1, 4, 16, 64), seed=5)
runs.append(("swap_narrow", s.optimize(2, 11, mode=bn.SWAP)[0][-1]["E_fixed"]))
s.eval_counts()
s.check()
s.close()
print("sanitize runs ok:", runs)
