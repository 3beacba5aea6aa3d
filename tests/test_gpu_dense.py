"""Dense MTTKRP / CP-ALS (BASELINE cfg 4 path) vs the reference's own
algorithm on a fully observed sparse tensor (the oracle the survey names for
this row: SPEC.md:127 -- the reference has no dense type).  Needs a B200."""

import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu


def _torch():
    import torch
    return torch


def rel(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return np.linalg.norm((a - b).ravel()) / np.linalg.norm(b.ravel())


def _dense_case(n, rank, seed):
    rng = np.random.default_rng(seed)
    dims = (n, n + 3, n + 5)
    X = rng.standard_normal(dims)
    fs = [rng.standard_normal((d, rank)) for d in dims]
    ot = O.OTensor(dims, np.arange(int(np.prod(dims)), dtype=np.uint64), X.ravel().copy())
    return X, fs, ot


@pytest.mark.parametrize("rank", [1, 8, 33, 64])
def test_dense_mttkrp_vs_fully_observed_oracle(rank):
    torch = _torch()
    from paper_1910_02371_b200.dense import dense_mttkrp
    X, fs, ot = _dense_case(40, rank, rank)
    Xd = torch.from_numpy(X).cuda()
    fd = [torch.from_numpy(f).cuda() for f in fs]
    for mode in range(3):
        got = dense_mttkrp(Xd, fd, mode).cpu().numpy()
        assert rel(got, O.mttkrp(ot, fs, mode)) < 1e-12


def test_dense_mttkrp_200cubed_rank64():
    torch = _torch()
    from paper_1910_02371_b200.dense import dense_mttkrp
    X, fs, ot = _dense_case(200, 64, 7)
    Xd = torch.from_numpy(X).cuda()
    fd = [torch.from_numpy(f).cuda() for f in fs]
    for mode in range(3):
        assert rel(dense_mttkrp(Xd, fd, mode).cpu().numpy(), O.mttkrp(ot, fs, mode)) < 1e-12


def test_dense_als_sweeps_match_sparse_reference_algorithm():
    torch = _torch()
    from paper_1910_02371_b200.dense import dense_als_sweep
    X, fs, ot = _dense_case(30, 16, 3)
    fd = [torch.from_numpy(f).cuda() for f in fs]
    ref = [f.copy() for f in fs]
    Xd = torch.from_numpy(X).cuda()
    for _ in range(2):
        dense_als_sweep(Xd, fd, 1e-5)
        O.als_sweep(ot, ref, 1e-5)
        for n in range(3):
            assert rel(fd[n].cpu().numpy(), ref[n]) < 1e-10


def test_dense_tf32_variant_accuracy_class():
    torch = _torch()
    from paper_1910_02371_b200.dense import dense_mttkrp
    X, fs, ot = _dense_case(60, 32, 11)
    Xd = torch.from_numpy(X).float().cuda()
    fd = [torch.from_numpy(f).float().cuda() for f in fs]
    for mode in range(3):
        got = dense_mttkrp(Xd, fd, mode).double().cpu().numpy()
        assert rel(got, O.mttkrp(ot, fs, mode)) < 5e-3  # TF32 products, fp32 sums
