"""GPU parity: the CUDA path (through the C-ABI) against the CPU oracle on identical seeded inputs.

Bar (north star): error vectors (counts) and u_p tiles bit-exact; accept/reject
sequences identical; exact fixed-point energies equal (which implies per-pass dE within 1e-9
relative and final E within 1e-6 relative of the oracle's fp64 sum, also asserted).
Sizes: the oracle finishes in seconds, shapes span several CTAs and a ragged tail (T not a
multiple of the 128-integrand padding); full BASELINE sizes are checked on sampled outputs.
"""
import numpy as np
import pytest

import synth  # noqa: E402

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def bn():
    import torch

    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device (run under gpurun)")
    from paper_2105_12620_b200 import bn as bnmod

    bnmod.load_library()
    return bnmod


def make(bn, oracle_mod, L, T, levels, tile_seed=1, bank_seed=2, sigma_s=1.0, radius=7, bank=None, U=None, form=0):
    a, b, px, py = bank if bank is not None else synth.make_bank(T, bank_seed)
    U = synth.make_tile(L, tile_seed) if U is None else U
    s = bn.Sampler(0)
    s.set_lattice(synth.D1, synth.D2, levels)
    s.set_bank(a, b, px, py)
    s.set_energy(2.1, sigma_s, radius)
    if form:
        s.set_energy_form(form)
    s.set_tile(L, U)
    o = oracle_mod.OracleProblem(L, len(a), tuple(levels), synth.D1, synth.D2, a, b, px, py,
                                 sigma_i=2.1, sigma_s=sigma_s, radius=radius, form=form)
    return s, o, U


# ----------------------------------------------------------------------------- counts / I_ref
@pytest.mark.parametrize("L,T,levels", [(16, 64, (16,)), (16, 200, (1, 4, 16, 64)), (32, 130, (4,)),
                                        (16, 1, (128,)), (64, 256, (4,))])
def test_counts_bit_exact(bn, oracle_mod, L, T, levels):
    s, o, U = make(bn, oracle_mod, L, T, levels)
    assert np.array_equal(s.eval_counts(), o.counts(U))


def test_counts_device_output_and_lattice_cut_bank(bn, oracle_mod):
    import torch

    N = 64
    bank = synth.axis_cut_bank(N, np.arange(N), "y")
    s, o, U = make(bn, oracle_mod, 16, N, (N,), bank=bank)
    out = torch.zeros((1, 256, N), dtype=torch.uint8, device="cuda")
    s.eval_counts(out)
    torch.cuda.synchronize()
    got = out.cpu().numpy()
    assert np.array_equal(got, o.counts(U))
    assert np.array_equal(got[0], np.broadcast_to(N - np.arange(N), (256, N)))  # exact integral


def test_references(bn, oracle_mod):
    s, o, _ = make(bn, oracle_mod, 16, 300, (16,))
    np.testing.assert_allclose(s.get_references(), o.references(), rtol=0, atol=1e-14)


# -------------------------------------------------------------------------------- energy
@pytest.mark.parametrize("L,T,levels,radius,sigma_s", [(16, 64, (16,), 7, 1.0), (32, 100, (1, 4, 16), 7, 1.0),
                                                       (32, 40, (4,), 3, 0.5), (16, 20, (64,), 1, 2.0)])
def test_energy_exact(bn, oracle_mod, L, T, levels, radius, sigma_s):
    s, o, U = make(bn, oracle_mod, L, T, levels, radius=radius, sigma_s=sigma_s)
    Ef, E = s.energy()
    Eo, Ep = o.energy(o.counts(U))
    assert Ef == Eo
    assert abs(E - Ep) <= 1e-9 * Ep


def test_energy_translation_invariance(bn, oracle_mod):
    s, o, U = make(bn, oracle_mod, 32, 50, (16,))
    Ef, _ = s.energy()
    s.set_tile(32, np.ascontiguousarray(np.roll(U.reshape(32, 32, 2), (5, 11), (0, 1)).reshape(-1, 2)))
    assert s.energy()[0] == Ef


# -------------------------------------------------------------------------- optimisation
def _check_run(s, o, U, passes, mode, seed, first_pass=0, K=1):
    st, lg = s.optimize(passes, seed, mode=mode, first_pass=first_pass, log=True, K=K)
    Uo, co, sto, lgo = o.optimize(U, mode=mode, passes=passes, first_pass=first_pass, seed=seed, log=True, K=K)
    assert np.array_equal(lg, lgo), "accept/reject sequence differs"
    assert np.array_equal(s.get_tile(), Uo), "tile differs"
    assert np.array_equal(s.eval_counts(), co), "counts differ"
    for g, r in zip(st, sto):
        assert g["accepted"] == r["accepted"] and g["proposed"] == r["proposed"]
        assert g["E_fixed"] == r["E_fixed"] and g["dE_sum"] == r["dE_sum"]
        assert abs(g["E"] - r["E_plain"]) <= 1e-6 * r["E_plain"]
    return st


@pytest.mark.parametrize("mode", [0, 1])
def test_c1_shape_full_run(bn, oracle_mod, mode):
    """C1: 16x16, 16 spp, T=64, greedy; 200 passes REDRAW (40 SWAP), compared pass by pass."""
    s, o, U = make(bn, oracle_mod, 16, 64, (16,))
    st = _check_run(s, o, U, 200 if mode == 0 else 40, mode, seed=3)
    assert st[-1]["E_fixed"] < st[0]["E_fixed"] + (-st[0]["dE_sum"])


@pytest.mark.parametrize("gather", ["", "nofuse"])
def test_c2_shape_swap(bn, oracle_mod, monkeypatch, gather):
    """C2 shape (SWAP, 4 spp) at 32x32, T=100 (ragged): commit fused with the next pass's partner
    gather (default), separate partner-map gather + commit (BN_FUSE=0)."""
    monkeypatch.setenv("BN_FUSE", "0" if gather == "nofuse" else "1")
    s, o, U = make(bn, oracle_mod, 32, 100, (4,))
    _check_run(s, o, U, 6, 1, seed=5)


def test_c3_shape_progressive(bn, oracle_mod):
    """C3 shape (1/4/16/64 progressive) at 32x32, T=130."""
    s, o, U = make(bn, oracle_mod, 32, 130, (1, 4, 16, 64))
    _check_run(s, o, U, 2, 0, seed=7)


@pytest.mark.parametrize("radius", [1, 4, 6])
def test_other_radii(bn, oracle_mod, radius):
    s, o, U = make(bn, oracle_mod, 16, 24, (4, 16), radius=radius)
    _check_run(s, o, U, 3, 0, seed=11)


def test_resume_and_determinism(bn, oracle_mod):
    s, o, U = make(bn, oracle_mod, 32, 40, (16,))
    s.optimize(2, 9)
    s.optimize(1, 9, first_pass=2)
    t1 = s.get_tile()
    s2, _, _ = make(bn, oracle_mod, 32, 40, (16,))
    s2.optimize(3, 9)
    assert np.array_equal(t1, s2.get_tile())


# ------------------------------------------------------------------------ argument errors
def test_errors(bn, oracle_mod):
    s = bn.Sampler(0)
    with pytest.raises(bn.BNError) as e:
        s.set_tile(16, np.zeros((256, 2), np.uint32))
    assert e.value.code == bn.BN_ESTATE
    with pytest.raises(bn.BNError) as e:
        s.set_lattice(1, 27, [4, 3])
    assert e.value.code == bn.BN_EINVAL
    s2, _, _ = make(bn, oracle_mod, 16, 8, (4,))
    with pytest.raises(bn.BNError) as e:
        s2.optimize(1, 1, K=2, mode=bn.SWAP)
    assert e.value.code == bn.BN_EINVAL
    with pytest.raises(bn.BNError) as e:
        s2.optimize(1, 1, K=9)
    assert e.value.code == bn.BN_EINVAL
    with pytest.raises(bn.BNError) as e:
        s2.set_tile(24, np.zeros((24 * 24, 2), np.uint32))
    assert e.value.code == bn.BN_EINVAL
    with pytest.raises(bn.BNError):
        s2.set_energy(2.1, 1.0, 8)


# ------------------------------------------------------------------ full BASELINE sizes
# complete passes at every BASELINE size: tests/test_gpu_fullsize.py (oracle goldens)


# ------------------------------------------------------------- bank-shard decomposition (C5)
@pytest.mark.parametrize("csplit", ["", "0"])
def test_window_distances_and_shard_decomposition(bn, oracle_mod, monkeypatch, csplit):
    """The multi-GPU (C5) exchange sums partial window distances over bank shards.  On one GPU:
    the full-bank distances equal the plain definition on the oracle's counts, and the shard
    contexts' partial distances (T split 3 ways, ragged) add up to them exactly.  Small tiles run
    one Gram item per neighbour chunk by default; BN_GRAM_CSPLIT=0 keeps whole items."""
    monkeypatch.setenv("BN_GRAM_CSPLIT", csplit)
    from paper_2105_12620_b200.dist import shard_range
    from tests.test_dist_cpu import _partial_distances

    L, T, levels = 32, 301, (4, 16)
    a, b, px, py = synth.make_bank(T, 21)
    U = synth.make_tile(L, 22)
    full, o, _ = make(bn, oracle_mod, L, T, levels, bank=(a, b, px, py), U=U)
    Df = full.window_distances()
    co = o.counts(U)
    for li in range(len(levels)):
        assert np.array_equal(Df[li], _partial_distances(co[li], L))
    acc = np.zeros_like(Df)
    for r in range(3):
        t0, t1 = shard_range(T, r, 3)
        s = bn.Sampler(0)
        s.set_lattice(synth.D1, synth.D2, levels)
        s.set_bank(a, b, px, py, t0, t1)
        s.set_energy(2.1, 1.0, 7)
        s.set_tile(L, U)
        assert np.array_equal(s.eval_counts(), co[:, :, t0:t1])
        acc += s.window_distances()
    assert np.array_equal(acc, Df)


def test_concurrent_contexts_match_sequential(bn, oracle_mod):
    """Independent pair tiles on their own streams, enqueued concurrently (the C4 bench layout),
    give bit-identical tiles to running each context alone."""
    import torch

    L, T, levels = 32, 96, (4, 16)
    runs = []
    for concurrent in (False, True):
        ctxs = []
        for j in range(3):
            st = torch.cuda.Stream()
            a, b, px, py = synth.make_bank(T, 40 + j)
            s = bn.Sampler(0, st.cuda_stream)
            s.set_lattice(synth.D1, synth.D2, levels)
            s.set_bank(a, b, px, py)
            s.set_energy(2.1, 1.0, 7)
            s.set_tile(L, synth.make_tile(L, 50 + j))
            ctxs.append(s)
        for j, s in enumerate(ctxs):
            s.optimize(4, 60 + j, stats=False)
            if not concurrent:
                torch.cuda.synchronize()
        torch.cuda.synchronize()
        runs.append([s.get_tile() for s in ctxs])
    for a_, b_ in zip(*runs):
        assert np.array_equal(a_, b_)


# ------------------------------------------------- window Gram, narrow row formats (f3)
@pytest.mark.parametrize("narrow", ["1", "e3m2", "u8", "0"])
@pytest.mark.parametrize("L,T,levels", [(16, 64, (16,)), (32, 300, (1, 4, 16, 64)), (64, 512, (4,)), (32, 130, (128,))])
def test_narrow_rows_window_distances(bn, oracle_mod, L, T, levels, narrow, monkeypatch):
    """The window Gram on every row format -- narrow e2m1 / e3m2 deltas chosen per level from the
    tile's range (1), e3m2 forced, the u8 layout through the narrow path, plain u8 rows (0) --
    gives the plain definition on the oracle's counts, after SWAP passes through the C-ABI equal to
    the oracle's (counts exported from the packed rows bit-exact)."""
    from tests.test_dist_cpu import _partial_distances

    monkeypatch.setenv("BN_NARROW", narrow)
    s, o, U = make(bn, oracle_mod, L, T, levels, tile_seed=32, bank_seed=31)
    _check_run(s, o, U, 2, 1, seed=13)
    co = s.eval_counts()
    D = s.window_distances()
    for li in range(len(levels)):
        assert np.array_equal(D[li], _partial_distances(co[li], L))


@pytest.mark.parametrize("narrow", ["1", "e3m2", "0"])
@pytest.mark.parametrize("mode", [0, 1])
def test_narrow_rows_mode_switches(bn, oracle_mod, monkeypatch, narrow, mode):
    """Mode switches across narrow and u8 rows: SWAP (packs), REDRAW (unpacks), SWAP again,
    against the oracle pass by pass (C3 shape, ragged T)."""
    monkeypatch.setenv("BN_NARROW", narrow)
    s, o, U = make(bn, oracle_mod, 32, 130, (1, 4, 16, 64))
    st, _ = s.optimize(2, 7, mode=mode, log=True)
    Uo, co, _, _ = o.optimize(U, mode=mode, passes=2, seed=7)
    assert np.array_equal(s.get_tile(), Uo)
    st, lg = s.optimize(2, 7, mode=1 - mode, first_pass=2, log=True)
    Uo, co, sto, lgo = o.optimize(Uo, co, mode=1 - mode, passes=2, first_pass=2, seed=7, log=True)
    assert np.array_equal(lg, lgo) and np.array_equal(s.get_tile(), Uo) and np.array_equal(s.eval_counts(), co)
    assert [x["E_fixed"] for x in st] == [x["E_fixed"] for x in sto]


@pytest.mark.parametrize("decide", ["", "flags", "per_class", "swap3"])
@pytest.mark.parametrize("L,mode", [(16, 0), (16, 1), (32, 1), (64, 1), (128, 0), (128, 1)])
def test_decide_kernels_parity(bn, oracle_mod, monkeypatch, decide, L, mode):
    """Every persistent decision kernel (register-prefetched cluster kernel = REDRAW default, SWAP
    per-member cluster kernel = SWAP default, one-warp-per-couple SWAP (swap3), cooperative flag
    kernel, per-class launches) against the oracle, both modes, 2 to 16 active indices per band."""
    monkeypatch.setenv("BN_DECIDE", decide)
    s, o, U = make(bn, oracle_mod, L, 40, (4, 16))
    _check_run(s, o, U, 2, mode, seed=21 + L + mode)


@pytest.mark.parametrize("rowflags", ["0", "1"])
def test_overlapped_passes_rowflags(bn, oracle_mod, monkeypatch, rowflags):
    """Multi-pass REDRAW with the next pass's counts prefetched on the low-priority stream; with
    BN_ROWFLAGS=1 the persistent Gram follows those counts row by row through device flags."""
    monkeypatch.setenv("BN_ROWFLAGS", rowflags)
    s, o, U = make(bn, oracle_mod, 32, 130, (1, 4, 16, 64))
    _check_run(s, o, U, 5, 0, seed=9)


# ------------------------------------------------------ paper-verbatim parallel swaps (f1)
def _check_paper_run(s, o, U, passes, seed, budget=None, first_pass=0, perm_seed=8):
    perm = synth.make_permutation(o.L * o.L, perm_seed)
    s.set_permutation(perm)
    b = budget or 0
    st, lg = s.optimize(passes, seed, mode=bn_mod().PAPER_SWAP, first_pass=first_pass, log=True, budget=b)
    Uo, co, sto, lgo = o.paper_optimize(U, perm, budget=budget, passes=passes, first_pass=first_pass, seed=seed,
                                        log=True)
    assert np.array_equal(lg, lgo), "accept/reject sequence differs"
    assert np.array_equal(s.get_tile(), Uo), "tile differs"
    assert np.array_equal(s.eval_counts(), co), "counts differ"
    for g, r in zip(st, sto):
        assert g["accepted"] == r["accepted"] and g["proposed"] == r["proposed"]
        assert g["E_fixed"] == r["E_fixed"] and g["dE_sum"] == r["dE_sum"]
        assert abs(g["E"] - r["E_plain"]) <= 1e-6 * r["E_plain"]
    return st


def bn_mod():
    from paper_2105_12620_b200 import bn as m

    return m


@pytest.mark.parametrize("L,T,levels,budget", [(16, 64, (16,), None), (16, 64, (16,), 2), (32, 130, (1, 4, 16), None),
                                               (64, 100, (4,), 2048), (32, 40, (4,), 1024)])
def test_paper_mode_parity(bn, oracle_mod, L, T, levels, budget):
    """Paper-verbatim snapshot couples (§3.4): accept flags, tiles, counts and the
    recomputed energies after every pass equal to the oracle (default N/4 budget, the
    single-couple degenerate case, the full budget P)."""
    s, o, U = make(bn, oracle_mod, L, T, levels)
    _check_paper_run(s, o, U, 6, seed=17, budget=budget)


def test_paper_mode_resume_and_errors(bn, oracle_mod):
    s, o, U = make(bn, oracle_mod, 32, 60, (4, 16))
    _check_paper_run(s, o, U, 3, seed=5, first_pass=4)
    s2, _, _ = make(bn, oracle_mod, 16, 8, (4,))
    with pytest.raises(bn.BNError) as e:                   # no permutation yet
        s2.optimize(1, 1, mode=bn.PAPER_SWAP)
    assert e.value.code == bn.BN_ESTATE
    with pytest.raises(bn.BNError) as e:                   # not a permutation
        s2.set_permutation(np.zeros(256, np.uint32))
    assert e.value.code == bn.BN_EINVAL
    s2.set_permutation(synth.make_permutation(256, 1))
    with pytest.raises(bn.BNError) as e:                   # odd budget
        s2.optimize(1, 1, mode=bn.PAPER_SWAP, budget=3)
    assert e.value.code == bn.BN_EINVAL


@pytest.mark.slow
def test_c2_full_size_paper_mode(bn, oracle_mod):
    """C2 tile (64x64, 4 spp, T=256) with the paper's own optimiser: 2 passes, N/4 budget."""
    cfg = synth.CONFIGS["C2"]
    U, bank = synth.problem_inputs(cfg)
    s, o, _ = make(bn, oracle_mod, cfg.L, cfg.T, cfg.levels, bank=bank, U=U)
    _check_paper_run(s, o, U, 2, seed=synth.opt_seed(cfg))


# ------------------------------------------------------------ Eq. 1 energy forms (f4)
@pytest.mark.parametrize("form", [1, 2])
@pytest.mark.parametrize("mode", [0, 1, 2])
def test_eq1_forms_parity(bn, oracle_mod, form, mode):
    """Eq. 1 as written (minimised) and maximised: energies and passes bit-exact in every mode."""
    s, o, U = make(bn, oracle_mod, 32, 100, (4, 16), form=form)
    assert s.energy()[0] == o.energy(o.counts(U))[0]
    if mode == 2:
        _check_paper_run(s, o, U, 3, seed=19)
    else:
        _check_run(s, o, U, 3, mode, seed=19)
    with pytest.raises(bn.BNError):
        s.set_energy_form(3)


# ----------------------------------------------------- evaluation criterion (f2, §3.3)
@pytest.mark.parametrize("L,T,levels,level", [(16, 40, (4, 16), 1), (32, 70, (16,), 0), (16, 33, (1, 4), 0)])
def test_eval_quality_parity(bn, oracle_mod, L, T, levels, level):
    """Denoised-RMSE curve (16 log-spaced sigmas in [0.25, 20], kernels larger than the tile wrap),
    error power spectrum and radial profile: the GPU's DFT/Parseval route against the oracle's plain
    convolution and plain DFT, fp64 (relative 1e-9 of the largest value)."""
    s, o, U = make(bn, oracle_mod, L, T, levels)
    sig = np.geomspace(0.25, 20.0, 16)
    r, S, prof = s.eval_quality(level, sig)
    c = o.counts(U)
    ro = o.denoised_rmse(c, level, sig)
    So, profo = o.error_spectrum(c, level)
    np.testing.assert_allclose(r, ro, rtol=1e-9, atol=1e-12)
    np.testing.assert_allclose(S, So, rtol=0, atol=1e-9 * So.max())
    np.testing.assert_allclose(prof, profo, rtol=1e-9, atol=1e-12 * profo.max())


def test_eval_quality_after_gpu_passes(bn, oracle_mod):
    """The criterion on GPU-optimised tiles (SWAP and paper mode) equals the oracle's on the same
    tile, and shows the paper's ordering: lower denoised RMSE than the random tile at sigma = 2."""
    s, o, U = make(bn, oracle_mod, 32, 48, (16,))
    r0, _, _ = s.eval_quality(0, [2.0], spectrum=False)
    s.optimize(6, 1, mode=1, stats=False)
    r1, S1, _ = s.eval_quality(0, [2.0])
    c1 = o.counts(s.get_tile())
    np.testing.assert_allclose(r1, o.denoised_rmse(c1, 0, [2.0]), rtol=1e-9)
    assert r1[0] < 0.8 * r0[0]
    with pytest.raises(bn.BNError):
        s.eval_quality(1, [2.0])
    with pytest.raises(bn.BNError):
        s.eval_quality(0, [0.0])


@pytest.mark.parametrize("L,T,levels,level,nb", [(16, 8, (16,), 0, 5), (32, 20, (4, 16, 64), 2, 12),
                                                  (64, 12, (16,), 0, 40)])
def test_eval_smooth_parity(bn, oracle_mod, L, T, levels, level, nb):
    """Smooth Gaussian-bump evaluation integrands (§3.5, f4): the GPU's denoised RMSE,
    spectrum and profile equal the oracle's plain per-sample estimates + convolution / DFT."""
    s, o, U = make(bn, oracle_mod, L, T, levels)
    bumps = synth.make_bumps(nb, L + nb)
    sig = [0.25, 1.0, 2.0, 6.0]
    r, S, prof, ref = s.eval_smooth(bumps, level, sig)
    e = o.smooth_errors(U, level, bumps)
    np.testing.assert_allclose(ref, [oracle_mod.bump_integral(*b) for b in bumps], rtol=1e-14)
    np.testing.assert_allclose(r, oracle_mod.denoised_rmse_images(e, sig), rtol=1e-9)
    So, po = oracle_mod.error_spectrum_images(e)
    np.testing.assert_allclose(S, So, rtol=1e-8, atol=1e-12 * So.max())
    np.testing.assert_allclose(prof, po, rtol=1e-8, atol=1e-12 * po.max())
    with pytest.raises(bn.BNError):
        s.eval_smooth(np.array([[0.5, 0.5, 0.0, 0.1]]), level, sig)


def test_eval_smooth_versatility_on_gpu_tiles(bn, oracle_mod):
    """PAPER.md §3.5: a tile optimised on Heavisides only (GPU SWAP passes) has lower low-frequency
    error power for the smooth family than the random tile (SPEC acceptance 8: <= 0.7x)."""
    s, o, U = make(bn, oracle_mod, 64, 64, (16,))
    bumps = synth.make_bumps(32, 3)
    _, _, p0, _ = s.eval_smooth(bumps, 0, [2.0])
    s.optimize(10, 2, mode=1, stats=False)
    _, _, p1, _ = s.eval_smooth(bumps, 0, [2.0])
    assert p1[:3].mean() <= 0.7 * p0[:3].mean()


@pytest.mark.parametrize("decide", ["", "notail", "nobig"])
@pytest.mark.parametrize("L,mode", [(256, 0), (256, 1), (512, 1)])
def test_decide_large_tiles(bn, oracle_mod, monkeypatch, decide, L, mode):
    """Tiles beyond one cluster's warps (L = 256, 512): SWAP through the fused pass tail with the
    bit-flag decisions (default), the bit-flag cluster kernel with several slots per warp (notail;
    REDRAW always), and with nobig the cooperative neighbour-band flag kernel (REDRAW) or the
    per-class launches (SWAP); full passes against the oracle (SWAP: 2, so the tail also gathers the
    next pass's candidates)."""
    monkeypatch.setenv("BN_DECIDE", "nobig" if decide == "nobig" else "")
    monkeypatch.setenv("BN_TAIL", "0" if decide == "notail" else "1")
    s, o, U = make(bn, oracle_mod, L, 16, (4,))
    _check_run(s, o, U, 2 if mode else 1, mode, seed=5 + L + mode)


# --------------------------------------------------------------- best-of-K REDRAW (f3, K > 1)
@pytest.mark.parametrize("L,T,levels,K,radius", [(16, 64, (16,), 2, 7), (32, 130, (1, 4, 16), 4, 7),
                                                 (16, 40, (4, 16), 8, 5), (64, 100, (4,), 3, 7)])
def test_best_of_k_parity(bn, oracle_mod, L, T, levels, K, radius):
    """Best-of-K re-draws (lowest exact dE of K Philox candidates, ties to the lowest j): accept
    logs, tiles, counts and exact energies equal to the oracle pass by pass."""
    s, o, U = make(bn, oracle_mod, L, T, levels, radius=radius)
    st = _check_run(s, o, U, 3, 0, seed=23, K=K)
    assert s.energy()[0] == st[-1]["E_fixed"]            # running energy == recomputed energy


def test_best_of_k_resume(bn, oracle_mod):
    s, o, U = make(bn, oracle_mod, 32, 48, (16,))
    s.optimize(2, 4, K=3, stats=False)
    _check_run(s, o, o.optimize(U, passes=2, seed=4, K=3)[0], 2, 0, seed=4, first_pass=2, K=3)


# ------------------------------------------------------------------------------- edge cases
def test_edge_cases_empty_and_degenerate(bn, oracle_mod):
    """Empty and degenerate inputs: T = 0 and out-of-range shards rejected; zero passes is a no-op;
    a constant tile (every error vector equal, every D = 0: the energy maximum) optimises exactly
    like the oracle; |a|, |b| beyond 2^15 rejected."""
    s = bn.Sampler(0)
    s.set_lattice(synth.D1, synth.D2, [16])
    with pytest.raises(bn.BNError) as e:
        s.set_bank(np.zeros(0, np.int32), np.zeros(0, np.int32), np.zeros(0, np.uint32), np.zeros(0, np.uint32))
    assert e.value.code == bn.BN_EINVAL
    a, b, px, py = synth.make_bank(8, 3)
    with pytest.raises(bn.BNError) as e:
        s.set_bank(a, b, px, py, 5, 5)
    assert e.value.code == bn.BN_EINVAL
    s.set_bank(a, b, px, py)
    with pytest.raises(bn.BNError) as e:  # beyond the largest parity-tested tile side (2048)
        s.set_tile(4096, np.zeros((4096 * 4096, 2), np.uint32))
    assert e.value.code == bn.BN_EINVAL
    with pytest.raises(bn.BNError) as e:
        s.set_bank(np.full(8, 1 << 16, np.int32), b, px, py)
    assert e.value.code == bn.BN_EINVAL
    U = np.tile(synth.make_tile(1, 4), (256, 1))
    s2, o, _ = make(bn, oracle_mod, 16, 24, (4, 16), U=U)
    E0 = s2.energy()[0]
    st, _ = s2.optimize(0, 1)
    assert st == [] and s2.energy()[0] == E0 and np.array_equal(s2.get_tile(), U)
    assert E0 == o.energy(o.counts(U))[0]
    for mode in (0, 1):
        s3, o3, _ = make(bn, oracle_mod, 16, 24, (4, 16), U=U)
        _check_run(s3, o3, U, 3, mode, seed=31)


def test_max_levels_and_spp(bn, oracle_mod):
    """Eight progressive levels up to the maximum 128 spp (uint8 counts reach 128), ragged T."""
    s, o, U = make(bn, oracle_mod, 16, 21, (1, 2, 4, 8, 16, 32, 64, 128))
    assert np.array_equal(s.eval_counts(), o.counts(U))
    _check_run(s, o, U, 2, 0, seed=33)
    _check_run(s, o, s.get_tile(), 2, 1, seed=34, first_pass=2)
