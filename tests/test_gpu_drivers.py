"""ALS / CCD++ / SGD sweeps and run() on the device vs the reference's golden
trajectories and the CPU oracle; device Philox sampling bit-exact vs the
reference.  Needs a B200 (``-m gpu``)."""

import numpy as np
import pytest

from conftest import golden
from oracle import oracle as O

import paper_1910_02371_b200 as cp
from paper_1910_02371_b200 import synth
from paper_1910_02371_b200.losses import get_loss, objective
from paper_1910_02371_b200.optim import (CompletionState, SolverConfig, als_sweep, ccd_sweep,
                                         init_state, run, sgd_sweep)

pytestmark = pytest.mark.gpu


def rel(a, b):
    a, b = np.asarray(a), np.asarray(b)
    s = np.linalg.norm(b.ravel())
    return np.linalg.norm((a - b).ravel()) / (s if s else 1.0)


def _cfg1():
    shape, keys, values, factors = synth.cfg1()
    return cp.SparseTensor(shape, keys, values), factors


def test_cfg1_als_five_sweeps_match_reference():
    z = golden("cfg1")
    t, factors = _cfg1()
    st = CompletionState(factors=[f.copy() for f in factors], rng=cp.RngState(0))
    cfg = SolverConfig(rank=10, reg=1e-5)
    for s in range(5):
        als_sweep(t, st, get_loss("ls"), cfg)
        for n in range(3):
            assert rel(st.factors[n], z[f"als{s}_f{n}"]) < 1e-10
        assert cp.rmse(t, st.factors) == pytest.approx(float(z[f"als{s}_rmse"]), rel=1e-10)
    assert rel(st.ls_gram[2][:5], z["als_gram2"]) < 1e-12
    assert rel(st.ls_rhs[2], z["als_rhs2"]) < 1e-12


def test_cfg1_ccd_two_sweeps_match_reference():
    z = golden("cfg1")
    t, factors = _cfg1()
    st = CompletionState(factors=[f.copy() for f in factors], rng=cp.RngState(0))
    cfg = SolverConfig(rank=10, reg=1e-5)
    for s in range(2):
        ccd_sweep(t, st, get_loss("ls"), cfg)
        for n in range(3):
            assert rel(st.factors[n], z[f"ccd{s}_f{n}"]) < 1e-10


def test_cfg1_sgd_three_steps_match_reference():
    z = golden("cfg1")
    t, factors = _cfg1()
    st = CompletionState(factors=[f.copy() for f in factors], rng=cp.RngState(0))
    cfg = SolverConfig(rank=10, reg=1e-4, step=1e-3, sample_rate=0.1, algorithm="sgd")
    for it in range(1, 4):
        sgd_sweep(t, st, get_loss("ls"), cfg, cp.RngState(11).child(1).child(it))
        for n in range(3):
            assert rel(st.factors[n], z[f"sgd{it}_f{n}"]) < 1e-12


def test_sample_bit_exact_vs_reference():
    z = golden("philox")
    keys = np.arange(10_000, dtype=np.uint64) * np.uint64(3)
    t = cp.SparseTensor((40_000,), keys, np.arange(10_000, dtype=np.float64))
    for j in range(int(z["n_sample"])):
        rng = cp.RngState(int(z[f"s{j}_seed"]), tuple(int(v) for v in z[f"s{j}_path"]))
        s = t.sample(float(z[f"s{j}_rate"]), rng)
        assert np.array_equal(s.keys, z[f"s{j}_keys"])
        assert np.array_equal(s.values, (s.keys // 3).astype(np.float64))


def test_sample_large_vs_oracle_and_shard_invariance():
    shape, keys, values, _ = synth.cfg2(nnz=2_000_003)
    t = cp.SparseTensor(shape, keys, values, validate=False)
    ot = O.OTensor(shape, keys, values)
    rng = cp.RngState(5, (1, 3))
    s = t.sample(0.01, rng)
    kept = O.sample_positions(ot, 0.01, 5, (1, 3))
    assert np.array_equal(s.keys, keys[kept])
    # shards with a global counter offset reproduce the single-device sample
    from paper_1910_02371_b200.sampling import sample_pattern
    cuts = [0, 1, 5, 999_999, 2_000_003]
    got = []
    for a, b in zip(cuts[:-1], cuts[1:]):
        part = cp.SparseTensor(shape, keys[a:b], values[a:b], validate=False)
        pat, parent = sample_pattern(part, 0.01, rng, counter_offset=a)
        got.append(parent.cpu().numpy().astype(np.int64) + a)
    assert np.array_equal(np.concatenate(got), kept)


def test_sample_rules():
    t = cp.build_tensor([((i, 0), float(i)) for i in range(10)], (10, 1))
    s = t.sample(1.0, cp.RngState(1))
    assert np.array_equal(s.keys, t.keys) and np.array_equal(s.values, t.values)
    assert cp.build_tensor([], (3, 3)).sample(0.5, cp.RngState(1)).nnz == 0
    for bad in (0.0, -0.1, 1.5):
        with pytest.raises(ValueError):
            t.sample(bad, cp.RngState(1))
    keys = np.arange(1000, dtype=np.uint64)
    t = cp.SparseTensor((1000,), keys, np.ones(1000))
    counts = [t.sample(0.1, cp.RngState(0).child(i)).nnz for i in range(300)]
    assert 90 <= np.mean(counts) <= 110


def test_drivers_small_run_traces_match_reference():
    z = golden("drivers_small")
    t = cp.SparseTensor(tuple(int(d) for d in z["dims"]), z["keys"], z["values"])
    for algo in ("als", "ccd", "sgd"):
        cfg = SolverConfig(rank=3, algorithm=algo, max_iters=4, seed=4, deterministic=True,
                           sample_rate=0.5, step=1e-3, record_every=1)
        trace, state = run(t, cfg, return_state=True)
        assert [r.iteration for r in trace.records] == list(z[f"{algo}_iters"])
        np.testing.assert_allclose([r.objective for r in trace.records], z[f"{algo}_obj"],
                                   rtol=1e-10)
        np.testing.assert_allclose([r.metric for r in trace.records], z[f"{algo}_metric"],
                                   rtol=1e-10)
        for n in range(3):
            assert rel(state.factors[n], z[f"{algo}_f{n}"]) < 1e-10


def _instance(rng, dims=(5, 4, 3), density=0.6):
    total = int(np.prod(dims))
    mask = rng.random(total) < density
    if not mask.any():
        mask[0] = True
    keys = np.flatnonzero(mask).astype(np.uint64)
    return cp.SparseTensor(dims, keys, rng.standard_normal(keys.size))


def test_als_monotone_and_fixed_point():
    rng = np.random.default_rng(0)
    loss = get_loss("ls")
    for trial in range(10):
        t = _instance(rng)
        cfg = SolverConfig(rank=2, reg=float(rng.random() * 0.1 + 1e-4), seed=trial)
        state = init_state(t, cfg, cp.RngState(trial).child(0))
        prev = objective(loss, t, state.factors, cfg.reg)
        for _ in range(3):
            als_sweep(t, state, loss, cfg)
            cur = objective(loss, t, state.factors, cfg.reg)
            assert cur <= prev * (1 + 1e-12)
            prev = cur
    t, truth = cp.gen_low_rank((6, 5, 4), 2, 1.0, rng=cp.RngState(1))
    state = CompletionState(factors=[f.copy() for f in truth], rng=cp.RngState(0))
    als_sweep(t, state, loss, SolverConfig(rank=2, reg=1e-10))
    for f, g in zip(state.factors, truth):
        assert np.allclose(f, g, atol=1e-6)


def test_ccd_rank1_equals_als_and_edge_rules():
    rng = np.random.default_rng(5)
    loss = get_loss("ls")
    for trial in range(10):
        t = _instance(rng)
        cfg = SolverConfig(rank=1, reg=float(rng.random() * 0.2 + 1e-6))
        sa = init_state(t, cfg, cp.RngState(trial).child(0))
        sc = CompletionState(factors=[f.copy() for f in sa.factors], rng=sa.rng)
        als_sweep(t, sa, loss, cfg)
        ccd_sweep(t, sc, loss, cfg)
        for a, c in zip(sa.factors, sc.factors):
            assert np.allclose(a, c, rtol=1e-12, atol=1e-12)
    t = cp.build_tensor([((0, 0, 0), 5.0)], (1, 1, 1))
    st = CompletionState(factors=[np.zeros((1, 1)), np.ones((1, 1)), np.ones((1, 1))],
                         rng=cp.RngState(0))
    ccd_sweep(t, st, loss, SolverConfig(rank=1, reg=0.0))
    assert st.factors[0][0, 0] == pytest.approx(5.0)
    t = cp.build_tensor([((0, 0, 0), 2.0)], (2, 1, 1))
    st = CompletionState(factors=[np.array([[0.5], [0.7]]), np.ones((1, 1)), np.ones((1, 1))],
                         rng=cp.RngState(0))
    ccd_sweep(t, st, loss, SolverConfig(rank=1, reg=0.0))
    assert st.factors[0][1, 0] == 0.7


def test_sgd_properties():
    rng = np.random.default_rng(8)
    loss = get_loss("ls")
    t = _instance(rng)
    cfg = SolverConfig(rank=2, algorithm="sgd", reg=1e-3, step=1e-9, sample_rate=1.0)
    st = init_state(t, cfg, cp.RngState(3).child(0))
    before = [f.copy() for f in st.factors]
    sgd_sweep(t, st, loss, cfg, cp.RngState(3).child(1))
    model = O.tttp(O.OTensor(t.shape, t.keys, np.ones(t.nnz)), before)
    phi1 = O.OTensor(t.shape, t.keys, 2.0 * (model - t.values))
    grads = [O.mttkrp(phi1, before, d) + 2e-3 * before[d] for d in range(3)]
    dot = sum(np.sum((a - b) * g) for a, b, g in zip(st.factors, before, grads))
    assert dot < 0.0
    t, truth = cp.gen_low_rank((5, 4, 3), 2, 1.0, rng=cp.RngState(9))
    st = CompletionState(factors=[f.copy() for f in truth], rng=cp.RngState(0))
    sgd_sweep(t, st, loss, SolverConfig(rank=2, algorithm="sgd", reg=0.0, step=1e-2),
              cp.RngState(1))
    for f, g in zip(st.factors, truth):
        assert np.allclose(f, g, atol=1e-12)
    t = _instance(np.random.default_rng(10))
    cfg = SolverConfig(rank=2, algorithm="sgd", step=1e-3, sample_rate=0.5, seed=3)
    a = run(t, cfg, return_state=True)[1].factors
    b = run(t, cfg, return_state=True)[1].factors
    for x, y in zip(a, b):
        assert np.array_equal(x, y)
    t = _instance(np.random.default_rng(11), dims=(6, 6, 6), density=0.9)
    t = t.with_values(t.values * 100.0)
    cfg = SolverConfig(rank=2, algorithm="sgd", step=10.0, sample_rate=1.0, max_iters=50,
                       record_every=1)
    with pytest.raises(cp.NumericalError):
        run(t, cfg)


def test_fast_ls_loss_identity():
    from paper_1910_02371_b200.losses import fast_ls_loss
    rng = np.random.default_rng(11)
    for _ in range(10):
        t = _instance(rng, dims=(6, 5, 4))
        factors = [rng.standard_normal((d, 3)) for d in t.shape]
        rhs = cp.mttkrp(t, factors, 0)
        new0, gram = cp.solve_factor(t.observation_mask(), factors, rhs, 0, reg=0.2,
                                     return_gram=True)
        factors[0] = new0
        fast = fast_ls_loss(float(np.sum(t.values ** 2)), new0, gram, rhs)
        direct = objective(get_loss("ls"), t, factors, reg=0.0)
        assert fast == pytest.approx(direct, rel=1e-10)
        # device tensors: batched symmetric mat-vec + fixed-order dots
        import torch
        fast_dev = fast_ls_loss(float(np.sum(t.values ** 2)), torch.from_numpy(new0).cuda(),
                                torch.from_numpy(gram).cuda(), torch.from_numpy(rhs).cuda())
        assert fast_dev == pytest.approx(fast, rel=1e-12)


def test_cfg2_scaled_sweeps_vs_oracle():
    # ALS / CCD++ / SGD on a 1e6-nonzero instance of the cfg 2 shape
    shape, keys, values, factors = synth.cfg2(nnz=1_000_000, rank=8)
    t = cp.SparseTensor(shape, keys, values, validate=False)
    ot = O.OTensor(shape, keys, values)
    fs = [f.copy() for f in factors]
    st = CompletionState(factors=[f.copy() for f in factors], rng=cp.RngState(0))
    als_sweep(t, st, get_loss("ls"), SolverConfig(rank=8, reg=1e-5))
    O.als_sweep(ot, fs, 1e-5)
    for n in range(3):
        assert rel(st.factors[n], fs[n]) < 1e-10
    fs = [f.copy() for f in factors]
    st = CompletionState(factors=[f.copy() for f in factors], rng=cp.RngState(0))
    ccd_sweep(t, st, get_loss("ls"), SolverConfig(rank=8, reg=1e-5))
    O.ccd_sweep(ot, fs, 1e-5)
    for n in range(3):
        assert rel(st.factors[n], fs[n]) < 1e-10
    fs = [f.copy() for f in factors]
    st = CompletionState(factors=[f.copy() for f in factors], rng=cp.RngState(0))
    cfg = SolverConfig(rank=8, reg=1e-4, step=1e-3, sample_rate=0.01, algorithm="sgd")
    sgd_sweep(t, st, get_loss("ls"), cfg, cp.RngState(7).child(1).child(1))
    O.sgd_sweep(ot, fs, 1e-4, 1e-3, 0.01, 7, (1, 1))
    for n in range(3):
        assert rel(st.factors[n], fs[n]) < 1e-10


@pytest.mark.parametrize("path", ["task", "flat", "lean"])
def test_ccd_kernel_paths_vs_oracle(path, monkeypatch):
    """Each CCD++ pass implementation (task table, flat segmented scan, and the
    memory-lean single canonical rhat read through the permutations) against
    the oracle on a Zipf-skewed cfg 3-shaped instance (long split rows, empty
    rows, a small mode), bitwise run-to-run deterministic."""
    from paper_1910_02371_b200 import optim
    if path == "lean":
        monkeypatch.setattr(optim, "_ccd_lean", lambda t: True)
    else:
        monkeypatch.setenv("CPFIT_CCD_PATH", path)
    shape, keys, values = synth.cfg3(nnz=400_000, shape=(48_019, 1_777, 218))
    rng = np.random.default_rng(4)
    factors = [rng.random((d, 6)) / np.sqrt(6) for d in shape]
    t = cp.SparseTensor(shape, keys, values, validate=False)
    ot = O.OTensor(shape, keys, values)
    fs = [f.copy() for f in factors]
    O.ccd_sweep(ot, fs, 1e-5)
    O.ccd_sweep(ot, fs, 1e-5)
    outs = []
    for _ in range(2):
        st = CompletionState(factors=[f.copy() for f in factors], rng=cp.RngState(0))
        ccd_sweep(t, st, get_loss("ls"), SolverConfig(rank=6, reg=1e-5))
        ccd_sweep(t, st, get_loss("ls"), SolverConfig(rank=6, reg=1e-5))
        outs.append(st.factors)
    for n in range(3):
        assert rel(outs[0][n], fs[n]) < 1e-10
        assert np.array_equal(outs[0][n], outs[1][n])


def test_init_laws_and_generators_match_reference():
    """init_state (uniform / gaussian / svd, calibrate_init) and the synthetic
    generators against tests/golden/init_state.npz (made by the reference:
    tests/golden/make_init_golden.py; optim.py:113-174, core.py:269-348)."""
    g = golden("init_state")
    shape = tuple(int(d) for d in g["shape"])
    t2, truth = cp.gen_low_rank(shape, 3, 0.4, "gaussian", cp.RngState(21).child(2))
    assert np.array_equal(t2.keys, g["keys"]) and np.array_equal(t2.values, g["values"])
    for k, f in enumerate(truth):
        assert np.array_equal(f, g[f"truth{k}"])
    ft = cp.gen_function_tensor((7, 8, 5), 0.5, cp.RngState(4))
    assert np.array_equal(ft.keys, g["func_keys"]) and np.array_equal(ft.values, g["func_values"])
    t = cp.SparseTensor(shape, g["keys"], g["values"])
    from paper_1910_02371_b200.optim import SolverConfig, init_state
    for init, rank, calib in [("uniform", 6, False), ("gaussian", 6, False), ("svd", 4, False),
                              ("svd", 12, False), ("uniform", 5, True), ("gaussian", 5, True)]:
        st = init_state(t, SolverConfig(rank=rank, init=init, seed=13, calibrate_init=calib))
        for k, f in enumerate(st.factors):
            want = g[f"{init}_{rank}_{int(calib)}_{k}"]
            if init != "svd" and not calib:
                assert np.array_equal(f, want), (init, rank, k)       # host draws: bit-exact
            else:  # svds vectors / the device TTTP inside the calibration
                np.testing.assert_allclose(f, want, rtol=1e-9, atol=1e-12)
