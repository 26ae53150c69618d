"""Complete passes at the full BASELINE sizes, through the C-ABI, against the CPU oracle.

The oracle's results for these runs take minutes of CPU time (C5: one SWAP pass of 65 536 pixels
x 224 neighbours x 8192 integrands), so they are precomputed by the committed script
`tests/golden/make_fullsize.py`, which calls only `oracle/` and `synth/` (never the CUDA path),
and stored in `tests/golden/fullsize_*.json`: per pass the exact E_fixed / dE_sum / accepted
count, the COMPLETE accept log (all 64 colour classes) and the sha256 of the tile; the sha256 of
the counts (error vectors) before and after.  Bar: everything bit-exact.

Runs use one bn_optimize call for all passes (the bench's launch configuration: SWAP passes end
with the fused commit + next-gather kernel, REDRAW passes prefetch the next pass's candidates on
the aux stream), the C4 pairs run concurrently on their own streams (the bench's C4 layout), and
the C5 run is repeated on a 1-rank NCCL communicator (the bank-shard exchange path).
"""
import hashlib

import numpy as np
import pytest

import synth
from tests.golden import make_bigtile
from tests.golden.make_fullsize import load, unpack_log

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.fixture(scope="module")
def bn():
    import torch

    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device (run under gpurun)")
    from paper_2105_12620_b200 import bn as bnmod

    bnmod.load_library()
    return bnmod


def _sampler(bn, g, stream=None):
    cfg = synth.CONFIGS[g["config"]]
    U, (a, b, px, py) = synth.problem_inputs(cfg, g["pair"])
    s = bn.Sampler(0, stream)
    s.set_lattice(synth.D1, synth.D2, cfg.levels)
    s.set_bank(a, b, px, py)
    s.set_energy(2.1, 1.0, 7)
    s.set_tile(cfg.L, U)
    return s


def _compare(s, g, st, lg):
    M = (g["L"] // 8) ** 2
    for pi, (got, ref) in enumerate(zip(st, g["per_pass"])):
        assert np.array_equal(lg[pi], unpack_log(ref["log_packbits_b64"], M)), f"pass {pi}: accept log differs"
        assert got["accepted"] == ref["accepted"] and got["proposed"] == ref["proposed"], f"pass {pi}"
        assert got["E_fixed"] == int(ref["E_fixed"]), f"pass {pi}: E_fixed differs"
        assert got["dE_sum"] == int(ref["dE_sum"]), f"pass {pi}: dE_sum differs"
        assert abs(got["E"] - ref["E_plain"]) <= 1e-6 * ref["E_plain"]   # north star: final E within 1e-6
    assert sha(s.get_tile()) == g["per_pass"][-1]["U_sha256"], "tile differs"
    assert sha(s.eval_counts()) == g["counts_final_sha256"], "counts (error vectors) differ"
    s.check()  # no device invariant failed in any launch


@pytest.mark.parametrize("job,narrow", [("C2_swap", "auto"), ("C3_swap", "auto"), ("C3_swap", "1"),
                                        ("C3_redraw", "auto")])
def test_full_passes_vs_oracle(bn, job, narrow, monkeypatch):
    """C2 (20 SWAP passes), C3 (2 SWAP passes, also on narrow rows; 2 REDRAW passes): every class of
    every pass."""
    monkeypatch.setenv("BN_NARROW", narrow)
    g = load(job)
    s = _sampler(bn, g)
    assert sha(s.eval_counts()) == g["counts0_sha256"], "initial counts differ"
    st, lg = s.optimize(g["passes"], g["seed"], mode=g["mode"], log=True)
    _compare(s, g, st, lg)
    s.close()


def test_c4_all_pairs_concurrent_vs_oracle(bn):
    """C4: all 8 independent dimension pairs, one SWAP pass each, enqueued concurrently on 8 streams."""
    import torch

    gs = [load(f"C4_pair{j}_swap") for j in range(8)]
    streams = [torch.cuda.Stream() for _ in gs]
    ss = [_sampler(bn, g, st.cuda_stream) for g, st in zip(gs, streams)]
    for s, g in zip(ss, gs):
        assert sha(s.eval_counts()) == g["counts0_sha256"]
    outs = [s.optimize(g["passes"], g["seed"], mode=g["mode"], log=True) for s, g in zip(ss, gs)]
    torch.cuda.synchronize()
    for s, g, (st, lg) in zip(ss, gs, outs):
        _compare(s, g, st, lg)
        s.close()


@pytest.mark.parametrize("comm", [False, True])
def test_c5_full_pass_vs_oracle(bn, comm):
    """C5 (256^2, T = 8192): one SWAP pass, all 64 classes of 1024 members; with `comm`, the context
    joins a 1-rank NCCL communicator, so the pass runs the bank-shard exchange (the in-place int32
    all-reduce of the window distances) exactly as each rank of a multi-GPU run does."""
    g = load("C5_swap")
    s = _sampler(bn, g)
    if comm:
        s.comm_init(bn.comm_unique_id(), 0, 1)
    assert sha(s.eval_counts()) == g["counts0_sha256"]
    st, lg = s.optimize(g["passes"], g["seed"], mode=g["mode"], log=True)
    _compare(s, g, st, lg)
    s.close()


def test_nccl_one_rank_small_runs_vs_oracle(bn, oracle_mod):
    """1-rank NCCL communicator on small shapes, both modes, several passes, against the live oracle
    (bn_comm_unique_id + bn_comm_init + the all-reduce in every pass and in bn_energy)."""
    for L, T, levels, mode in [(32, 100, (4, 16), 1), (32, 64, (16,), 0)]:
        a, b, px, py = synth.make_bank(T, 2)
        U = synth.make_tile(L, 1)
        s = bn.Sampler(0)
        s.set_lattice(synth.D1, synth.D2, levels)
        s.set_bank(a, b, px, py)
        s.set_energy(2.1, 1.0, 7)
        s.set_tile(L, U)
        s.comm_init(bn.comm_unique_id(), 0, 1)
        o = oracle_mod.OracleProblem(L, T, levels, synth.D1, synth.D2, a, b, px, py)
        assert s.energy()[0] == o.energy(o.counts(U))[0]
        st, lg = s.optimize(3, 5, mode=mode, log=True)
        Uo, co, sto, lgo = o.optimize(U, mode=mode, passes=3, seed=5, log=True)
        assert np.array_equal(lg, lgo) and np.array_equal(s.get_tile(), Uo)
        assert [x["E_fixed"] for x in st] == [x["E_fixed"] for x in sto]
        s.close()


@pytest.mark.parametrize("name", sorted(make_bigtile.JOBS))
def test_largest_tiles_vs_oracle(bn, name):
    """The largest tiles the API accepts (L = 1024, 2048; T = 8, 4 spp): one REDRAW and one SWAP
    pass (the cooperative band-flag decisions / per-class launches beyond one cluster) against
    oracle goldens: counts before and after, the accept log of all 64 classes, the tile, E_fixed
    and dE_sum, all bit-exact."""
    g = make_bigtile.load(name)
    U, (a, b, px, py) = make_bigtile.inputs(g["L"])
    s = bn.Sampler(0)
    s.set_lattice(synth.D1, synth.D2, g["levels"])
    s.set_bank(a, b, px, py)
    s.set_energy(2.1, 1.0, 7)
    s.set_tile(g["L"], U)
    assert sha(s.eval_counts()) == g["counts0_sha256"]
    st, lg = s.optimize(1, g["seed"], mode=g["mode"], log=True)
    assert sha(np.asarray(lg[0], np.uint8)) == g["log_sha256"], "accept log differs"
    assert st[0]["accepted"] == g["accepted"] and st[0]["proposed"] == g["proposed"]
    assert st[0]["E_fixed"] == int(g["E_fixed"]) and st[0]["dE_sum"] == int(g["dE_sum"])
    assert sha(s.get_tile()) == g["U_sha256"], "tile differs"
    assert sha(s.eval_counts()) == g["counts_final_sha256"], "counts differ"
    s.check()
    s.close()
