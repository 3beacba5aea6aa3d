"""Generalized (Poisson log-link) losses on the device vs the reference's own
outputs (tests/golden/generalized.npz, made by tests/golden/make_golden.py):
derivative tensors and objective with exp-clamp counting, inner-Newton ALS
(also with frozen curvature) and CCD++ sweeps, SGD steps, run() traces, and
least squares through the generalized ALS path.  SURVEY 8(f) rank 2."""

import numpy as np
import pytest

from conftest import golden

import paper_1910_02371_b200 as cp
from paper_1910_02371_b200 import losses as Lz
from paper_1910_02371_b200.optim import (CompletionState, SolverConfig, als_sweep, ccd_sweep,
                                         run, sgd_sweep)

pytestmark = pytest.mark.gpu


def rel(a, b):
    a, b = np.asarray(a), np.asarray(b)
    s = np.linalg.norm(b.ravel())
    return np.linalg.norm((a - b).ravel()) / (s if s else 1.0)


def _data():
    z = golden("generalized")
    t = cp.SparseTensor(tuple(int(d) for d in z["dims"]), z["keys"], z["values"])
    init = [z[f"init{n}"] for n in range(3)]
    return z, t, init


def test_poisson_derivatives_objective_and_clamp_counts():
    z, t, init = _data()
    loss = cp.get_loss("poisson")
    big = [z["big0"], init[1], init[2]]
    model = cp.model_at_observed(t.observation_mask(), big)
    p1, p2 = cp.derivative_tensors(loss, t, model)
    assert rel(p1.values, z["clamp_phi1"]) < 1e-12
    assert rel(p2.values, z["clamp_phi2"]) < 1e-12
    assert loss.diagnostics["exp_clamped"] == int(z["clamp_count_derivs"])
    obj = cp.objective(loss, t, big, reg=1e-3)
    assert obj == pytest.approx(float(z["clamp_obj"]), rel=1e-12)
    assert loss.diagnostics["exp_clamped"] == int(z["clamp_count_total"])
    # the fused TTTP loss epilogue gives the same tensors
    import torch
    F = [torch.from_numpy(f).cuda() for f in big]
    d1, d2, n = Lz.device_derivatives(loss, t, F)
    assert rel(d1.cpu().numpy(), z["clamp_phi1"]) < 1e-12
    assert rel(d2.cpu().numpy(), z["clamp_phi2"]) < 1e-12
    assert 2 * n == int(z["clamp_count_derivs"])


@pytest.mark.parametrize("algo", ["als", "als_frozen", "ccd", "sgd"])
def test_poisson_sweeps_match_reference(algo):
    z, t, init = _data()
    kw = {"als_frozen": {"freeze_curvature": True},
          "sgd": {"sample_rate": 0.5, "step": 1e-2}}.get(algo, {})
    loss = cp.get_loss("poisson")
    cfg = SolverConfig(rank=3, reg=1e-3, loss="poisson", **kw)
    st = CompletionState(factors=[f.copy() for f in init], rng=cp.RngState(0))
    nsweep = 3 if algo == "sgd" else 2
    for s in range(nsweep):
        if algo.startswith("als"):
            als_sweep(t, st, loss, cfg)
        elif algo == "ccd":
            ccd_sweep(t, st, loss, cfg)
        else:
            sgd_sweep(t, st, loss, cfg, cp.RngState(5).child(s))
        for n in range(3):
            assert isinstance(st.factors[n], np.ndarray)
            assert rel(st.factors[n], z[f"{algo}{s}_f{n}"]) < 1e-10, (algo, s, n)


def test_least_squares_through_generalized_als():
    z, t, init = _data()
    tl = t.with_values(z["lsgen_values"])
    st = CompletionState(factors=[f.copy() for f in init], rng=cp.RngState(0))
    als_sweep(tl, st, cp.get_loss("ls"), SolverConfig(rank=3, reg=1e-3), generalized=True)
    for n in range(3):
        assert rel(st.factors[n], z[f"lsgen_f{n}"]) < 1e-10


def test_user_registered_loss_keeps_host_callables():
    """A loss registered by the user (no device evaluator) runs its numpy
    callables like the reference; with least-squares math it reproduces the
    generalized least-squares sweep."""
    z, t, init = _data()
    base = Lz.least_squares()
    Lz.register_loss("ls_user", lambda: Lz.LossFunction(
        ident="ls_user", phi=base.phi, dphi=base.dphi, d2phi=base.d2phi))
    loss = cp.get_loss("ls_user")
    assert loss.device_id is None
    tl = t.with_values(z["lsgen_values"])
    st = CompletionState(factors=[f.copy() for f in init], rng=cp.RngState(0))
    als_sweep(tl, st, loss, SolverConfig(rank=3, reg=1e-3))
    for n in range(3):
        assert rel(st.factors[n], z[f"lsgen_f{n}"]) < 1e-10


@pytest.mark.parametrize("algo", ["als", "ccd", "sgd"])
def test_poisson_run_traces(algo):
    z, t, init = _data()
    cfg = SolverConfig(rank=3, algorithm=algo, loss="poisson", max_iters=3, seed=4,
                       deterministic=True, record_every=1, sample_rate=0.5, step=1e-2)
    trace, state = run(t, cfg, return_state=True)
    obj = np.array([r.objective for r in trace.records])
    met = np.array([r.metric for r in trace.records])
    assert rel(obj, z[f"run_{algo}_obj"]) < 1e-10
    assert rel(met, z[f"run_{algo}_metric"]) < 1e-10
    for n in range(3):
        assert rel(state.factors[n], z[f"run_{algo}_f{n}"]) < 1e-9


def test_poisson_sgd_fp32_device_factors_close_to_fp64():
    """fp32 CUDA factors select the fp32 kernels (TTTP loss epilogue, MTTKRP,
    SGD update); one Poisson SGD step stays within 1e-4 of the fp64 step."""
    import torch
    z, t, init = _data()
    loss = cp.get_loss("poisson")
    cfg = SolverConfig(rank=3, reg=1e-3, loss="poisson", sample_rate=0.5, step=1e-2)
    st64 = CompletionState(factors=[f.copy() for f in init], rng=cp.RngState(0))
    sgd_sweep(t, st64, loss, cfg, cp.RngState(5).child(0))
    st32 = CompletionState(factors=[torch.from_numpy(f).float().cuda() for f in init],
                           rng=cp.RngState(0))
    sgd_sweep(t, st32, cp.get_loss("poisson"), cfg, cp.RngState(5).child(0))
    for n in range(3):
        assert st32.factors[n].dtype == torch.float32
        assert rel(st32.factors[n].double().cpu().numpy(), st64.factors[n]) < 1e-4
