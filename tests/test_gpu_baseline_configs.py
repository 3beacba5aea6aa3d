"""Parity at the BASELINE configurations' real shapes and precisions
(VERDICT r1 "next round" item 1), on identical bytes for GPU and oracle:

* cfg 3 at full size (480,189 x 17,770 x 2,182, 100,480,507 Zipf nonzeros,
  R = 32, lambda = 1e-5): one ALS sweep and one CCD++ sweep from the same
  init_state draws, GPU vs the oracle's C restatement on the box's host
  cores (optim.py:180-268), factors within 1e-10;
* cfg 5 shape and dtype (order 4, 1e5 x 1e5 x 1e5 x 1e3, fp32, R = 64) at
  1e7 nonzeros: the TTTP residual norm within 1e-4 of the fp64 oracle on the
  fp32-rounded inputs, one SGD step (rate 0.01, step 1e-3, lambda 1e-4) with
  a bit-exact Philox sample, gradients within 1e-4 and the post-step
  residual norm within 1e-4 (optim.py:300-330, core.py:173-183).
cfg 4 at 800^3 is in test_gpu_dense.py.  Needs a B200 and ~40 GB of host RAM.
"""

import os

import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu


def _torch():
    import torch
    return torch


def rel(a, b):
    a, b = np.asarray(a, dtype=np.float64), np.asarray(b, dtype=np.float64)
    return float(np.linalg.norm((a - b).ravel()) / np.linalg.norm(b.ravel()))


@pytest.fixture(scope="module")
def cfg3():
    torch = _torch()
    import paper_1910_02371_b200 as cp
    from paper_1910_02371_b200 import synth
    shape, keys, vals = synth.cfg3_device()
    keys_h = keys.cpu().numpy().view(np.uint64)
    vals_h = vals.cpu().numpy()
    t = cp.SparseTensor.from_device(shape, keys, vals)
    del keys, vals
    ot = O.OTensor(shape, keys_h, vals_h)
    O.set_threads(os.cpu_count() or 1)
    init = O.init_factors(shape, 32, 0, (0,))
    yield shape, t, ot, init
    del t
    torch.cuda.empty_cache()


def test_cfg3_full_size_als_sweep_vs_oracle(cfg3):
    torch = _torch()
    from paper_1910_02371_b200.optim import _als_ls_device
    shape, t, ot, init = cfg3
    assert t.nnz == 100_480_507
    F = [torch.from_numpy(f).cuda() for f in init]
    _als_ls_device(t, F, 1e-5)
    ref = [f.copy() for f in init]
    O.als_sweep(ot, ref, 1e-5)
    for n in range(3):
        assert rel(F[n].cpu().numpy(), ref[n]) < 1e-10, n


def test_cfg3_full_size_ccd_sweep_vs_oracle(cfg3):
    torch = _torch()
    from paper_1910_02371_b200.optim import _ccd_ls_device
    shape, t, ot, init = cfg3
    F = [torch.from_numpy(f).cuda() for f in init]
    _ccd_ls_device(t, F, 1e-5)
    ref = [f.copy() for f in init]
    O.ccd_sweep(ot, ref, 1e-5)
    for n in range(3):
        assert rel(F[n].cpu().numpy(), ref[n]) < 1e-10, n


def test_cfg5_shape_fp32_residual_and_sgd_step():
    torch = _torch()
    import paper_1910_02371_b200 as cp
    from paper_1910_02371_b200 import synth
    from paper_1910_02371_b200.losses import tttp_affine
    from paper_1910_02371_b200.optim import _sgd_apply_device, _sgd_grads_device
    O.set_threads(os.cpu_count() or 1)
    nnz = 10_000_000
    shape, t0, values, F = synth.cfg5_device(nnz=nnz, with_keys=False)
    t = t0.with_values(values)  # fp32 values = rank-8 model + N(0, 0.1)
    assert t.order == 4 and t.nnz == nnz and F[0].dtype == torch.float32 and F[0].shape[1] == 64
    keys_h = t.keys
    vals64 = values.cpu().numpy().astype(np.float64)
    f64 = [f.cpu().numpy().astype(np.float64) for f in F]
    ot = O.OTensor(shape, keys_h, vals64)

    # TTTP residual t - model in fp32 vs the fp64 oracle on the same (fp32) inputs
    resid = tttp_affine(t, F, -1.0, 1.0, torch.float32).cpu().numpy().astype(np.float64)
    ref_resid = vals64 - O.tttp(ot.with_values(np.ones(nnz)), f64)
    assert abs(np.linalg.norm(resid) - np.linalg.norm(ref_resid)) / np.linalg.norm(ref_resid) < 1e-4
    assert rel(resid, ref_resid) < 1e-4

    # one SGD step: the Bernoulli(0.01) sample is bit-exact, gradients within 1e-4
    rate, step, reg = 0.01, 1e-3, 1e-4
    rng = cp.RngState(5).child(1).child(1)
    sampled = t.sample(rate, rng)
    kept = O.sample_positions(ot, rate, 5, (1, 1))
    assert np.array_equal(sampled.keys, keys_h[kept])
    grads, n = _sgd_grads_device(t, F, rate, rng, torch.float32)
    assert n == kept.size
    s = O.OTensor(shape, keys_h[kept], vals64[kept])
    model = O.tttp(s.with_values(np.ones(s.nnz)), f64)
    phi1 = s.with_values(2.0 * (model - s.values))
    for mode in range(4):
        assert rel(grads[mode].cpu().numpy(), O.mttkrp(phi1, f64, mode)) < 1e-4, mode
    _sgd_apply_device(F, grads, step, 2.0 * step * reg * rate)
    ref = [f.copy() for f in f64]
    O.sgd_sweep(ot, ref, reg, step, rate, 5, (1, 1))
    resid = tttp_affine(t, F, -1.0, 1.0, torch.float32).cpu().numpy().astype(np.float64)
    ref_resid = vals64 - O.tttp(ot.with_values(np.ones(nnz)), ref)
    assert abs(np.linalg.norm(resid) - np.linalg.norm(ref_resid)) / np.linalg.norm(ref_resid) < 1e-4
    for mode in range(4):
        assert rel(F[mode].cpu().numpy(), ref[mode]) < 1e-4, mode
