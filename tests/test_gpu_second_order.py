"""Gauss-Newton / Newton on the device (cpfit_tttp_subst + MTTKRP + Gram +
solve_rows + PCG) vs vectors produced by the reference itself
(tests/golden/second_order.npz) and the reference's property tests
(tests/test_optim.py:251-436).  Needs a B200 (``-m gpu``)."""

import numpy as np
import pytest

from conftest import golden

import paper_1910_02371_b200 as cp
from paper_1910_02371_b200 import NumericalError
from paper_1910_02371_b200.optim import CompletionState, SolverConfig

pytestmark = pytest.mark.gpu


def rel(a, b):
    a, b = np.asarray(a), np.asarray(b)
    s = np.linalg.norm(b.ravel())
    return np.linalg.norm((a - b).ravel()) / (s if s else 1.0)


def _case(z, c):
    dims = tuple(int(d) for d in z[f"hv{c}_dims"])
    keys = np.arange(int(np.prod(dims)), dtype=np.uint64)
    t = cp.SparseTensor(dims, keys, z[f"hv{c}_vals"])
    n = len(dims)
    return (t, [z[f"hv{c}_f{k}"] for k in range(n)], [z[f"hv{c}_x{k}"] for k in range(n)],
            str(z[f"hv{c}_ident"]), str(z[f"hv{c}_variant"]), float(z[f"hv{c}_reg"]))


def test_hessian_matvec_and_gradient_match_reference():
    z = golden("second_order")
    for c in range(int(z["hv_cases"])):
        t, fs, xs, ident, variant, reg = _case(z, c)
        loss = cp.get_loss(ident)
        model = cp.model_at_observed(t.observation_mask(), fs)
        phi1, phi2 = cp.derivative_tensors(loss, t, model)
        y = cp.hessian_matvec(phi1, phi2, fs, xs, variant=variant, reg=reg)
        g = cp.gradient_blocks(t, fs, loss, reg)
        for k in range(len(fs)):
            assert rel(y[k], z[f"hv{c}_y{k}"]) < 1e-12, (c, k)
            assert rel(g[k], z[f"hv{c}_g{k}"]) < 1e-12, (c, k)


def test_hessian_linear_and_self_adjoint():
    z = golden("second_order")
    t, fs, xs, ident, _, _ = _case(z, 0)
    loss = cp.get_loss(ident)
    phi1, phi2 = cp.derivative_tensors(loss, t, cp.model_at_observed(t.observation_mask(), fs))
    out = cp.hessian_matvec(phi1, phi2, fs, [np.zeros_like(f) for f in fs], reg=0.5)
    assert all(np.all(b == 0.0) for b in out)
    rng = np.random.default_rng(15)
    for variant in ("gauss_newton", "newton"):
        x1 = [rng.standard_normal(f.shape) for f in fs]
        x2 = [rng.standard_normal(f.shape) for f in fs]
        y1 = cp.hessian_matvec(phi1, phi2, fs, x1, variant=variant, reg=0.3)
        y2 = cp.hessian_matvec(phi1, phi2, fs, x2, variant=variant, reg=0.3)
        lhs = sum(np.sum(a * b) for a, b in zip(y1, x2))
        rhs = sum(np.sum(a * b) for a, b in zip(x1, y2))
        assert lhs == pytest.approx(rhs, rel=1e-12)
    with pytest.raises(ValueError):
        cp.hessian_matvec(phi1, phi2, fs, xs, variant="bogus")
    with pytest.raises(ValueError):
        cp.hessian_matvec(phi1, phi2, fs, xs[:-1])


def test_gn_step_trajectories_match_reference():
    z = golden("second_order")
    dims = tuple(int(d) for d in z["gn_dims"])
    t = cp.SparseTensor(dims, z["gn_keys"], z["gn_values"])
    for tag, variant, kw in (("gnls", "gauss_newton", {}), ("ntls", "newton", {}),
                             ("gnls_damped", "gauss_newton", {"gn_damping": 0.1})):
        cfg = SolverConfig(rank=3, reg=1e-4, cg_tol=1e-10, cg_max=300, **kw)
        st = CompletionState(factors=[z[f"gn_init{n}"].copy() for n in range(3)],
                             rng=cp.RngState(0))
        for s in range(3):
            used = cp.gn_step(t, st, cp.get_loss("ls"), cfg, variant=variant)
            ref_cg = int(z[f"{tag}_cg"][s])
            assert abs(used - ref_cg) <= max(3, ref_cg // 10), (tag, s, used, ref_cg)
            for n in range(3):
                assert rel(st.factors[n], z[f"{tag}{s}_f{n}"]) < 1e-8, (tag, s, n)
    tp = t.with_values(z["gnpo_values"])
    cfg = SolverConfig(rank=3, reg=1e-3, cg_tol=1e-10, cg_max=300, loss="poisson")
    st = CompletionState(factors=[z[f"gnpo_init{n}"].copy() for n in range(3)],
                         rng=cp.RngState(0))
    for s in range(2):
        used = cp.gn_step(tp, st, cp.get_loss("poisson"), cfg)
        assert abs(used - int(z["gnpo_cg"][s])) <= max(3, int(z["gnpo_cg"][s]) // 10)
        for n in range(3):
            assert rel(st.factors[n], z[f"gnpo{s}_f{n}"]) < 1e-8


def test_run_gn_newton_traces_match_reference():
    z = golden("second_order")
    rng2 = np.random.default_rng(26)
    dims = (8, 7, 6)
    total = int(np.prod(dims))
    mask = rng2.random(total) < 0.5
    keys = np.flatnonzero(mask).astype(np.uint64)
    t = cp.SparseTensor(dims, keys, rng2.standard_normal(keys.size))
    for algo, kw in (("gn", {"calibrate_init": True, "gn_damping": 1.0}),
                     ("newton", {"warmup_sweeps": 1, "gn_damping": 1.0,
                                 "calibrate_init": True})):
        cfg = SolverConfig(rank=3, algorithm=algo, max_iters=3, seed=4, deterministic=True,
                           record_every=1, **kw)
        trace, state = cp.run(t, cfg, return_state=True)
        assert [r.iteration for r in trace.records] == list(z[f"run_{algo}_iters"])
        np.testing.assert_allclose([r.objective for r in trace.records], z[f"run_{algo}_obj"],
                                   rtol=1e-8)
        np.testing.assert_allclose([r.metric for r in trace.records], z[f"run_{algo}_metric"],
                                   rtol=1e-8)
        for n in range(3):
            assert rel(state.factors[n], z[f"run_{algo}_f{n}"]) < 1e-7


def test_gn_properties():
    # gradient norm drop near a solution (tests/test_optim.py:387-400)
    t, truth = cp.gen_low_rank((8, 7, 6), 2, 1.0, rng=cp.RngState(21))
    noise = np.random.default_rng(0)
    fs = [f + 0.01 * noise.standard_normal(f.shape) for f in truth]
    loss = cp.get_loss("ls")
    cfg = SolverConfig(rank=2, reg=1e-9, cg_tol=1e-6, cg_max=200)
    st = CompletionState(factors=fs, rng=cp.RngState(0))

    def gnorm():
        return np.linalg.norm(np.concatenate([g.ravel() for g in cp.gradient_blocks(
            t, st.factors, loss, cfg.reg)]))
    before = gnorm()
    cp.gn_step(t, st, loss, cfg)
    assert gnorm() < before / 10
    # zero factors are a fixed point for least squares
    st = CompletionState(factors=[np.zeros((d, 2)) for d in t.shape], rng=cp.RngState(0))
    cp.gn_step(t, st, loss, SolverConfig(rank=2, reg=0.0))
    assert all(np.allclose(f, 0.0, atol=1e-14) for f in st.factors)
    # non-convex loss rejected
    bad = cp.LossFunction(ident="bad", phi=lambda tv, m: -m ** 2, dphi=lambda tv, m: -2 * m,
                          d2phi=lambda tv, m: np.full_like(np.asarray(m), -2.0))
    st = CompletionState(factors=[f.copy() for f in truth], rng=cp.RngState(0))
    with pytest.raises(NumericalError):
        cp.gn_step(t, st, bad, SolverConfig(rank=2))


def test_gn_device_resident_factors():
    import torch
    z = golden("second_order")
    dims = tuple(int(d) for d in z["gn_dims"])
    t = cp.SparseTensor(dims, z["gn_keys"], z["gn_values"])
    cfg = SolverConfig(rank=3, reg=1e-4, cg_tol=1e-10, cg_max=300)
    st = CompletionState(factors=[torch.from_numpy(z[f"gn_init{n}"].copy()).cuda()
                                  for n in range(3)], rng=cp.RngState(0))
    cp.gn_step(t, st, cp.get_loss("ls"), cfg)
    assert all(f.is_cuda for f in st.factors)
    for n in range(3):
        assert rel(st.factors[n].cpu().numpy(), z[f"gnls0_f{n}"]) < 1e-8


def test_singular_preconditioner_raises():
    # reg = 0 and a mode-0 row without entries: (G_i + 0 I) = 0 is singular,
    # like np.linalg.solve in the reference's BlockDiagPreconditioner.apply
    keys = np.array([k for k in range(4 * 3 * 3)], dtype=np.uint64)
    t = cp.SparseTensor((5, 3, 3), keys, np.random.default_rng(1).standard_normal(keys.size))
    fs = [np.random.default_rng(2 + n).standard_normal((d, 2)) for n, d in enumerate(t.shape)]
    st = CompletionState(factors=fs, rng=cp.RngState(0))
    with pytest.raises(NumericalError, match="singular block-diagonal preconditioner"):
        cp.gn_step(t, st, cp.get_loss("ls"), SolverConfig(rank=2, reg=0.0))
    pre = cp.BlockDiagPreconditioner(t.with_values(np.full(t.nnz, 2.0)), fs, 0.0)
    with pytest.raises(NumericalError):
        pre.apply([np.ones_like(f) for f in fs])
