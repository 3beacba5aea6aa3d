"""PCG and gauge rebalancing of the second-order step on plain numpy blocks
(no device work): the reference's TestPcg / rebalance tests
(tests/test_optim.py:340-386, 413-424)."""

import numpy as np
import pytest

import paper_1910_02371_b200 as cp
from paper_1910_02371_b200 import NumericalError


def test_pcg_identity_system():
    b = [np.ones((3, 2)), np.full((2, 2), 2.0)]
    x, iters = cp.pcg_solve(lambda v: [vi.copy() for vi in v],
                            lambda v: [vi.copy() for vi in v], b, rel_tol=1e-8, max_iters=10)
    assert iters == 1
    for xi, bi in zip(x, b):
        assert np.allclose(xi, bi)


def test_pcg_random_spd_vs_direct():
    rng = np.random.default_rng(19)
    for _ in range(20):
        n = int(rng.integers(3, 30))
        a = rng.standard_normal((n, n))
        spd = a @ a.T + n * np.eye(n)
        b = rng.standard_normal((n, 1))
        x, _ = cp.pcg_solve(lambda v: [spd @ v[0]], lambda v: [vi.copy() for vi in v], [b],
                            rel_tol=1e-8, max_iters=300)
        ref = np.linalg.solve(spd, b)
        assert np.linalg.norm(x[0] - ref) / np.linalg.norm(ref) < 1e-7


def test_pcg_perfect_preconditioner():
    rng = np.random.default_rng(20)
    n = 12
    a = rng.standard_normal((n, n))
    spd = a @ a.T + n * np.eye(n)
    inv = np.linalg.inv(spd)
    b = rng.standard_normal((n, 1))
    _, iters = cp.pcg_solve(lambda v: [spd @ v[0]], lambda v: [inv @ v[0]], [b],
                            rel_tol=1e-10, max_iters=50)
    assert iters == 1


def test_pcg_zero_rhs_and_nonfinite():
    x, iters = cp.pcg_solve(lambda v: v, lambda v: v, [np.zeros((4, 2))], rel_tol=1e-3,
                            max_iters=5)
    assert iters == 0 and np.all(x[0] == 0.0)
    with pytest.raises(NumericalError):
        cp.pcg_solve(lambda v: [v[0] * np.nan], lambda v: v, [np.ones((2, 1))], 1e-3, 5)
    with pytest.raises(ValueError):
        cp.pcg_solve(lambda v: v, lambda v: v, [np.ones((2, 1))], 1.5, 5)


def test_rebalance_equalizes_norms():
    rng = np.random.default_rng(23)
    fs = [rng.standard_normal((d, 2)) for d in (4, 3, 3)]
    fs[0] *= 100.0
    before = np.einsum("ir,jr,kr->ijk", *fs)
    cp.rebalance_factors(fs)
    after = np.einsum("ir,jr,kr->ijk", *fs)
    assert np.allclose(before, after, rtol=1e-12)
    norms = np.stack([np.linalg.norm(f, axis=0) for f in fs])
    assert np.allclose(norms[0], norms[1], rtol=1e-12)
