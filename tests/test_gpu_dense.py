"""Dense MTTKRP / CP-ALS (BASELINE cfg 4 path) vs the reference's own
algorithm on a fully observed sparse tensor (the oracle the survey names for
this row: SPEC.md:127 -- the reference has no dense type), and at the full
800^3 size against host numpy (einsum('ijk,jr,kr->ir') through BLAS).
Needs a B200."""

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


def _dense_case(dims, rank, seed):
    rng = np.random.default_rng(seed)
    X = rng.standard_normal(dims)
    fs = [rng.standard_normal((d, rank)) for d in dims]
    ot = O.OTensor(dims, np.arange(int(np.prod(dims)), dtype=np.uint64), X.ravel().copy())
    return X, fs, ot


# (40, 43, 45): K odd -> rows not 16-byte aligned -> the kernels' non-TMA path;
# (40, 42, 44) / (36, 40, 52): TMA path with partial tiles and partial K chunks
@pytest.mark.parametrize("dims", [(40, 43, 45), (40, 42, 44), (36, 40, 52)])
@pytest.mark.parametrize("rank", [1, 8, 33, 64, 100])
def test_dense_mttkrp_vs_fully_observed_oracle(dims, rank):
    torch = _torch()
    from paper_1910_02371_b200.dense import dense_mttkrp
    X, fs, ot = _dense_case(dims, rank, rank)
    Xd = torch.from_numpy(X).cuda()
    fd = [torch.from_numpy(f).cuda() for f in fs]
    for mode in range(3):
        got = dense_mttkrp(Xd, fd, mode).cpu().numpy()
        assert rel(got, O.mttkrp(ot, fs, mode)) < 1e-12


def test_dense_mttkrp_200cubed_rank64():
    torch = _torch()
    from paper_1910_02371_b200.dense import dense_mttkrp
    X, fs, ot = _dense_case((200, 200, 200), 64, 7)
    Xd = torch.from_numpy(X).cuda()
    fd = [torch.from_numpy(f).cuda() for f in fs]
    for mode in range(3):
        assert rel(dense_mttkrp(Xd, fd, mode).cpu().numpy(), O.mttkrp(ot, fs, mode)) < 1e-12
    # the slot of the output mode is ignored (may be None)
    got = dense_mttkrp(Xd, [None, fd[1], fd[2]], 0).cpu().numpy()
    assert rel(got, O.mttkrp(ot, fs, 0)) < 1e-12


def test_dense_mttkrp_deterministic():
    torch = _torch()
    from paper_1910_02371_b200.dense import dense_mttkrp
    X, fs, _ = _dense_case((96, 80, 64), 64, 5)
    Xd = torch.from_numpy(X).cuda()
    fd = [torch.from_numpy(f).cuda() for f in fs]
    for mode in range(3):
        a = dense_mttkrp(Xd, fd, mode)
        b = dense_mttkrp(Xd, fd, mode)
        assert torch.equal(a, b)


def _host_mttkrp(X, fs, mode):
    """einsum('ijk,jr,kr->ir') and analogues on the host, through BLAS."""
    I, J, K = X.shape
    A, B, C = fs
    if mode == 0:
        T = (X.reshape(I * J, K) @ C).reshape(I, J, -1)
        return np.einsum("ijr,jr->ir", T, B)
    if mode == 1:
        T = (X.reshape(I * J, K) @ C).reshape(I, J, -1)
        return np.einsum("ijr,ir->jr", T, A)
    KR = (A[:, None, :] * B[None, :, :]).reshape(I * J, -1)
    return X.reshape(I * J, K).T @ KR


def test_dense_mttkrp_800cubed_vs_host_einsum():
    """BASELINE cfg 4 at full size: 800^3 fp64 N(0,1), R = 64."""
    torch = _torch()
    from paper_1910_02371_b200.dense import dense_mttkrp
    g = torch.Generator(device="cuda")
    g.manual_seed(4)
    n, R = 800, 64
    Xd = torch.randn((n, n, n), generator=g, dtype=torch.float64, device="cuda")
    fd = [torch.randn((n, R), generator=g, dtype=torch.float64, device="cuda") for _ in range(3)]
    X = Xd.cpu().numpy()
    fs = [f.cpu().numpy() for f in fd]
    for mode in range(3):
        ref = _host_mttkrp(X, fs, mode)
        got = dense_mttkrp(Xd, fd, mode).cpu().numpy()
        assert rel(got, ref) < 1e-12, mode
        # and the TF32 tensor-core variant on the fp32-rounded inputs
        got32 = dense_mttkrp(Xd.float(), [f.float() for f in fd], mode).double().cpu().numpy()
        assert rel(got32, ref) < 5e-3, mode


def test_dense_xc_and_gram():
    torch = _torch()
    from paper_1910_02371_b200.dense import gram_hadamard, xc_product
    X, fs, _ = _dense_case((50, 60, 70), 24, 9)
    Xd = torch.from_numpy(X).cuda()
    T = xc_product(Xd, torch.from_numpy(fs[2]).cuda()).cpu().numpy()
    assert rel(T, np.einsum("ijk,kr->ijr", X, fs[2])) < 1e-13
    G = gram_hadamard([torch.from_numpy(f).cuda() for f in fs[:2]]).cpu().numpy()
    assert rel(G, (fs[0].T @ fs[0]) * (fs[1].T @ fs[1])) < 1e-13


def test_dense_als_sweeps_match_sparse_reference_algorithm():
    torch = _torch()
    from paper_1910_02371_b200.dense import dense_als_sweep
    X, fs, ot = _dense_case((30, 33, 36), 16, 3)
    fd = [torch.from_numpy(f).cuda() for f in fs]
    ref = [f.copy() for f in fs]
    Xd = torch.from_numpy(X).cuda()
    for _ in range(2):
        dense_als_sweep(Xd, fd, 1e-5)
        O.als_sweep(ot, ref, 1e-5)
        for n in range(3):
            assert rel(fd[n].cpu().numpy(), ref[n]) < 1e-10


@pytest.mark.parametrize("dims", [(60, 64, 68), (130, 96, 200), (40, 43, 45)])
def test_dense_tf32_variant_accuracy_class(dims):
    torch = _torch()
    from paper_1910_02371_b200.dense import dense_mttkrp
    X, fs, ot = _dense_case(dims, 32, 11)
    Xd = torch.from_numpy(X).float().cuda()
    fd = [torch.from_numpy(f).float().cuda() for f in fs]
    for mode in range(3):
        got = dense_mttkrp(Xd, fd, mode).double().cpu().numpy()
        assert rel(got, O.mttkrp(ot, fs, mode)) < 5e-3  # TF32 products, fp32 sums


def test_dense_rejects_bad_arguments():
    torch = _torch()
    from paper_1910_02371_b200.dense import dense_mttkrp
    Xd = torch.zeros((4, 5, 6), dtype=torch.float64, device="cuda")
    f = [torch.zeros((d, 3), dtype=torch.float64, device="cuda") for d in (4, 5, 6)]
    with pytest.raises(ValueError):
        dense_mttkrp(Xd, f, 3)
    with pytest.raises(ValueError):
        dense_mttkrp(Xd, [f[0], f[1][:, :2], f[2]], 0)
    with pytest.raises(ValueError):
        dense_mttkrp(Xd, [f[0], None, f[2]], 0)


def test_dense_shared_solve_and_singular_fallback():
    torch = _torch()
    from paper_1910_02371_b200.dense import solve_shared
    from paper_1910_02371_b200.exceptions import NumericalError
    rng = np.random.default_rng(2)
    B = rng.standard_normal((50, 24))
    G = B.T @ B
    rhs = rng.standard_normal((77, 24))
    x = solve_shared(torch.from_numpy(G).cuda(), torch.from_numpy(rhs).cuda(), 1e-3).cpu().numpy()
    ref = np.linalg.solve(G + 1e-3 * np.eye(24), rhs.T).T
    assert rel(x, ref) < 1e-12
    # not SPD -> the per-row path with the reference's singular-row semantics
    with pytest.raises(NumericalError):
        solve_shared(torch.zeros((24, 24), dtype=torch.float64, device="cuda"),
                     torch.from_numpy(rhs).cuda(), 0.0)
