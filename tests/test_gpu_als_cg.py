"""Implicit-CG ALS (BASELINE cfg 3 "ALS completion with implicit CG"): the
Gram-free row product cpfit_gram_matvec against the oracle's Gram blocks, and
the per-row CG mode update / sweep against the oracle's direct ALS sweep (the
reference solves each row with LAPACK, kernels.py:259; CG has no reference
counterpart, so agreement is to the CG tolerance).  Needs a B200 (``-m gpu``)."""

import numpy as np
import pytest

from oracle import oracle as O

import paper_1910_02371_b200 as cp
from paper_1910_02371_b200 import synth
from paper_1910_02371_b200.losses import get_loss
from paper_1910_02371_b200.optim import CompletionState, SolverConfig, als_sweep

pytestmark = pytest.mark.gpu


def rel(a, b):
    a, b = np.asarray(a, dtype=np.float64), np.asarray(b, dtype=np.float64)
    s = np.linalg.norm(b.ravel())
    return np.linalg.norm((a - b).ravel()) / (s if s else 1.0)


def _random_instance(rng, dims, nnz):
    total = int(np.prod(dims))
    keys = np.sort(rng.choice(total, size=min(nnz, total), replace=False)).astype(np.uint64)
    return keys, rng.random(keys.size) + 0.1


@pytest.mark.parametrize("dims,rank", [((7, 6, 5), 3), ((40, 30, 20), 10), ((50, 9, 33), 16),
                                       ((30, 20, 10, 6), 8), ((25, 40), 32), ((12, 9, 8), 40)])
def test_gram_matvec_vs_oracle_gram(dims, rank):
    rng = np.random.default_rng(sum(dims) + rank)
    keys, w = _random_instance(rng, dims, int(np.prod(dims) * 0.3))
    wt = cp.SparseTensor(dims, keys, w)
    ow = O.OTensor(dims, keys, w)
    factors = [rng.standard_normal((d, rank)) for d in dims]
    for mode in range(len(dims)):
        x = rng.standard_normal((dims[mode], rank))
        want = np.einsum("irs,is->ir", O.gram_blocks(ow, factors, mode), x)
        got = cp.gram_matvec(wt, factors, x, mode)
        assert rel(got, want) < 1e-12
        # unit weights through the observation mask; inactive rows return 0
        active = (rng.random(dims[mode]) < 0.6).astype(np.int32)
        want1 = np.einsum("irs,is->ir",
                          O.gram_blocks(ow.with_values(np.ones(ow.nnz)), factors, mode), x)
        got1 = cp.gram_matvec(wt.observation_mask(), factors, x, mode, row_active=active)
        assert rel(got1, want1 * active[:, None]) < 1e-12
        assert not got1[active == 0].any()


def test_gram_matvec_fp32_and_split_rows():
    import torch
    # Zipf rows long enough to be split into several tasks (deterministic combine)
    shape, keys, values = synth.cfg3(nnz=300_000, shape=(4_801, 1_777, 218))
    t = cp.SparseTensor(shape, keys, values, validate=False)
    ot = O.OTensor(shape, keys, np.ones(keys.size))
    rng = np.random.default_rng(3)
    rank = 16
    factors = [rng.random((d, rank)) / np.sqrt(rank) for d in shape]
    for mode in (0, 1, 2):
        x = rng.standard_normal((shape[mode], rank))
        want = np.einsum("irs,is->ir", O.gram_blocks(ot, factors, mode), x)
        mask = t.observation_mask()
        got = cp.gram_matvec(mask, factors, x, mode)
        assert rel(got, want) < 1e-12
        assert np.array_equal(got, cp.gram_matvec(mask, factors, x, mode))  # run-to-run bitwise
        f32 = [torch.from_numpy(f).cuda().float() for f in factors]
        got32 = cp.gram_matvec(mask, f32, torch.from_numpy(x).cuda().float(), mode)
        assert got32.dtype == torch.float32
        assert rel(got32.double().cpu().numpy(), want) < 1e-4


def test_cg_als_sweep_matches_direct_oracle_cfg1():
    shape, keys, values, factors = synth.cfg1()
    t = cp.SparseTensor(shape, keys, values)
    ot = O.OTensor(shape, keys, values)
    fs = [f.copy() for f in factors]
    st = CompletionState(factors=[f.copy() for f in factors], rng=cp.RngState(0))
    cfg = SolverConfig(rank=10, reg=1e-5, als_solver="cg", cg_tol=1e-13, cg_max=60)
    for sweep in range(2):
        als_sweep(t, st, get_loss("ls"), cfg)
        O.als_sweep(ot, fs, 1e-5)
        for n in range(3):
            assert rel(st.factors[n], fs[n]) < 1e-8
        assert st.ls_gram[0] is None and st.ls_rhs[0] is not None


def test_cg_als_default_tolerance_residuals_and_skew():
    """cfg 3-shaped Zipf instance: with the default cg_tol every row's residual
    satisfies ||b_i - (G_i + reg I) x_i|| <= cg_tol ||b_i|| (or the row hit
    cg_max); the sweep lowers the objective like the direct sweep does."""
    from paper_1910_02371_b200.optim import _als_mode_cg_device, _to_dev_factors
    shape, keys, values = synth.cfg3(nnz=400_000, shape=(48_019, 1_777, 218))
    t = cp.SparseTensor(shape, keys, values, validate=False)
    ot = O.OTensor(shape, keys, values)
    rng = np.random.default_rng(5)
    rank, reg, tol = 8, 1e-5, 5e-3
    factors = [rng.random((d, rank)) / np.sqrt(rank) for d in shape]
    F = _to_dev_factors([f.copy() for f in factors])
    for mode in range(3):
        x, rhs, iters = _als_mode_cg_device(t, F, mode, reg, tol, 3 * rank)
        assert 1 <= iters <= 3 * rank
        xh, bh = x.cpu().numpy(), rhs.cpu().numpy()
        G = O.gram_blocks(ot.with_values(np.ones(ot.nnz)), [f.cpu().numpy() for f in F], mode)
        res = bh - (np.einsum("irs,is->ir", G, xh) + reg * xh)
        rn, bn = np.linalg.norm(res, axis=1), np.linalg.norm(bh, axis=1)
        assert np.all(rn <= tol * bn * (1 + 1e-9) + 1e-300)
        assert not xh[bn == 0].any()  # rows without entries: x = 0
        F[mode] = x
    direct = [f.copy() for f in factors]
    O.als_sweep(ot, direct, reg)
    got = cp.rmse(t, [f.cpu().numpy() for f in F])
    want = O.rmse(ot, direct)
    assert got <= want * 1.05


def test_cg_als_run_driver_and_validation():
    with pytest.raises(ValueError):
        SolverConfig(als_solver="qr")
    shape, keys, values, _ = synth.cfg1()
    t = cp.SparseTensor(shape, keys, values)
    a = cp.run(t, SolverConfig(rank=5, reg=1e-5, max_iters=4, seed=1))
    b = cp.run(t, SolverConfig(rank=5, reg=1e-5, max_iters=4, seed=1, als_solver="cg",
                               cg_tol=1e-12, cg_max=40))
    assert len(a.records) == len(b.records)
    assert np.allclose([r.metric for r in a.records], [r.metric for r in b.records], rtol=1e-7)
    assert np.allclose([r.objective for r in a.records], [r.objective for r in b.records],
                       rtol=1e-7)


@pytest.mark.parametrize("rank", [16, 32])
def test_fragment_gram_rank16_32_zipf_vs_oracle(rank):
    """The register-fragment Gram kernel at the ranks of cfg 2 / cfg 3 on a
    Zipf instance with split rows: unit and weighted Grams and one ALS sweep
    (fused right-hand side) against the oracle."""
    shape, keys, values = synth.cfg3(nnz=200_000, shape=(4_801, 1_777, 218))
    t = cp.SparseTensor(shape, keys, values, validate=False)
    ot = O.OTensor(shape, keys, values)
    rng = np.random.default_rng(rank)
    factors = [rng.random((d, rank)) / np.sqrt(rank) for d in shape]
    for mode in range(3):
        got = cp.gram_blocks(t.observation_mask(), factors, mode)
        want = O.gram_blocks(ot.with_values(np.ones(ot.nnz)), factors, mode)
        assert rel(got, want) < 1e-12
        gw = cp.gram_blocks(t, factors, mode)  # weighted (sqrt(w) precomputed)
        assert rel(gw, O.gram_blocks(ot, factors, mode)) < 1e-12
    st = CompletionState(factors=[f.copy() for f in factors], rng=cp.RngState(0))
    als_sweep(t, st, get_loss("ls"), SolverConfig(rank=rank, reg=1e-2))
    fs = [f.copy() for f in factors]
    O.als_sweep(ot, fs, 1e-2)
    for n in range(3):
        assert rel(st.factors[n], fs[n]) < 1e-10
