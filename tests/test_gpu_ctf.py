"""ctf-style façade == its mapping
onto the package's kernels, bit for bit (same device kernels).  Needs a B200."""

import numpy as np
import pytest

import paper_1910_02371_b200 as cp
from paper_1910_02371_b200 import ctf
from oracle import oracle as O

pytestmark = pytest.mark.gpu


def _case(seed=1, shape=(30, 40, 50), density=0.05, R=6):
    rng = np.random.default_rng(seed)
    T = ctf.tensor(shape, sp=True)
    T.fill_sp_random(-1.0, 1.0, density, seed=seed)
    U, V, W = (rng.standard_normal((d, R)) for d in shape)
    return T, U, V, W


def test_tensor_construction_and_write():
    T = ctf.tensor((4, 5, 6), sp=True)
    assert T.sparse.nnz == 0
    T.write((np.array([3, 0, 3]), np.array([1, 2, 1]), np.array([5, 0, 5])),
            np.array([1.0, 2.0, 4.0]))  # duplicate summed
    keys, vals = T.read_all()
    assert keys.tolist() == [0 * 30 + 2 * 6 + 0, 3 * 30 + 1 * 6 + 5]
    assert vals.tolist() == [2.0, 5.0]
    D = ctf.tensor((3, 4))
    assert D.read_all().shape == (3, 4) and not D.sp


def test_tttp_matches_kernel():
    T, U, V, W = _case()
    Omega = ctf.getOmega(T)
    S = ctf.TTTP(Omega, [U, V, W])
    ref = cp.tttp(T.sparse.observation_mask(), [U, V, W])
    assert np.array_equal(S.sparse.values, ref.values)
    S2 = ctf.TTTP(Omega, [U, None, W])
    assert np.array_equal(S2.sparse.values, cp.tttp(T.sparse.observation_mask(), [U, None, W]).values)
    # residual R = T - TTTP(Omega, [U, V, W])
    R = T - S
    assert np.array_equal(R.sparse.values, T.sparse.values - ref.values)
    ot = O.OTensor(T.shape, T.sparse.keys, np.ones(T.sparse.nnz))
    assert np.allclose(S.sparse.values, O.tttp(ot, [U, V, W]), rtol=1e-13, atol=1e-13)


def test_mttkrp_solve_factor_in_place():
    T, U, V, W = _case(2)
    rhs = np.zeros_like(U)
    ctf.MTTKRP(T, [rhs, V, W], 0)
    assert np.array_equal(rhs, cp.mttkrp(T.sparse, [None, V, W], 0))
    Omega = ctf.getOmega(T)
    U2 = np.zeros_like(U)
    ctf.Solve_Factor(Omega, [U2, V, W], rhs, 0, 1e-3)
    ref = cp.solve_factor(T.sparse.observation_mask(), [None, V, W], rhs, 0, reg=1e-3)
    assert np.array_equal(U2, ref)
    # dense Tensor operands are written in place too
    rt = ctf.tensor(U.shape)
    ctf.MTTKRP(T, [rt, ctf.Tensor.from_array(V), W], 0)
    assert np.array_equal(rt.read_all(), rhs)


def test_einsum_patterns():
    T, U, V, W = _case(3)
    assert np.array_equal(ctf.einsum("ijk,jr,kr->ir", T, V, W),
                          cp.mttkrp(T.sparse, [None, V, W], 0))
    assert np.array_equal(ctf.einsum("ijk,ir,jr->kr", T, U, V),
                          cp.mttkrp(T.sparse, [U, V, None], 2))
    r = 2
    a = ctf.einsum("ijk,j,k->i", T, V[:, r], W[:, r])
    assert np.array_equal(a, cp.mttkrp(T.sparse, [None, V[:, r:r + 1], W[:, r:r + 1]], 0)[:, 0])
    Omega = ctf.getOmega(T)
    b = ctf.einsum("ijk,j,j,k,k->i", Omega, V[:, r], V[:, r], W[:, r], W[:, r])
    vv, ww = (V[:, r] * V[:, r])[:, None], (W[:, r] * W[:, r])[:, None]
    assert np.array_equal(b, cp.mttkrp(Omega.sparse, [None, vv, ww], 0)[:, 0])
    with pytest.raises(ValueError):
        ctf.einsum("ir,jr,kr->ijk", U, V, W)


def test_einsum_dense_cuda_operand():
    import torch
    from paper_1910_02371_b200.dense import dense_mttkrp
    rng = np.random.default_rng(4)
    X = torch.from_numpy(rng.standard_normal((20, 24, 28))).cuda()
    B = torch.from_numpy(rng.standard_normal((24, 5))).cuda()
    C = torch.from_numpy(rng.standard_normal((28, 5))).cuda()
    got = ctf.einsum("ijk,jr,kr->ir", X, B, C)
    assert torch.equal(got, dense_mttkrp(X, [None, B, C], 0))


def test_sample_in_place_matches_sparse_tensor_sample():
    T, *_ = _case(5, density=0.2)
    ref = T.sparse.sample(0.3, cp.RngState(9))
    T2 = T.copy()
    T2.sample(0.3, cp.RngState(9))
    assert np.array_equal(T2.sparse.keys, ref.keys)
    assert np.array_equal(T2.sparse.values, ref.values)
