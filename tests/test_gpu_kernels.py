"""Parity of the CUDA kernels (called through the C-ABI) with the reference's
golden vectors and with the CPU oracle.  Needs a B200 (``-m gpu``).

Tolerances (north_star): indexing/sorting bit-exact; fp64 within 1e-10
relative (tighter where the reference's own tests are tighter); fp32 within
1e-4 relative on the residual norm.
"""

import numpy as np
import pytest

from conftest import golden
from oracle import oracle as O

import paper_1910_02371_b200 as cp
from paper_1910_02371_b200 import synth

pytestmark = pytest.mark.gpu


def _torch():
    import torch
    return torch


def rel(a, b):
    a = np.asarray(a)
    b = np.asarray(b)
    d = np.linalg.norm((a - b).ravel())
    s = np.linalg.norm(b.ravel())
    return d / s if s else d


def _case(z, c):
    p = f"c{c}_"
    dims = tuple(int(d) for d in z[p + "dims"])
    factors = [z[p + f"f{n}"] for n in range(len(dims))]
    t = cp.SparseTensor(dims, z[p + "keys"], z[p + "values"])
    return p, dims, factors, t


# --------------------------------------------------------------------------
# golden vectors from the reference

def test_small_cases_match_reference_goldens():
    z = golden("kernels_small")
    for c in range(int(z["n_cases"])):
        p, dims, factors, t = _case(z, c)
        mode = int(z[p + "mode"])
        absent = int(z[p + "absent"])
        tf = list(factors)
        if absent >= 0:
            tf[absent] = None
        got = cp.tttp(t, tf)
        np.testing.assert_allclose(got.values, z[p + "tttp"], rtol=1e-12, atol=1e-12)
        np.testing.assert_allclose(cp.mttkrp(t, factors, mode), z[p + "mttkrp"],
                                   rtol=1e-12, atol=1e-12)
        w = t.with_values(np.abs(t.values) + 0.1)
        np.testing.assert_allclose(cp.gram_blocks(w, factors, mode), z[p + "gram"],
                                   rtol=1e-12, atol=1e-12)
        x = cp.solve_factor(w, factors, z[p + "rhs"], mode, reg=float(z[p + "reg"]))
        np.testing.assert_allclose(x, z[p + "solve"], rtol=1e-10, atol=1e-10)
        perm, offsets = cp.counting_sort_by_mode(t, mode)
        assert np.array_equal(perm, z[p + "perm"])
        assert np.array_equal(offsets, z[p + "offsets"])


def test_layout_goldens_bit_exact():
    z = golden("layout")
    dims2 = tuple(int(d) for d in z["cs_dims"])
    t = cp.SparseTensor(dims2, z["cs_keys"], np.ones(z["cs_keys"].size))
    for mode in range(3):
        perm, offsets = t.mode_group(mode)
        assert np.array_equal(perm, z[f"cs_perm{mode}"])
        assert np.array_equal(offsets, z[f"cs_offsets{mode}"])
    dims3 = tuple(int(d) for d in z["dl_dims"])
    t3 = cp.SparseTensor(dims3, z["dl_keys"], np.ones(z["dl_keys"].size))
    assert np.array_equal(np.stack(t3.coords()), z["dl_coords"])


def test_cfg1_matches_reference():
    z = golden("cfg1")
    shape, keys, values, factors = synth.cfg1()
    t = cp.SparseTensor(shape, keys, values)
    out = cp.tttp(t, factors).values
    assert rel(out, z["tttp"]) < 1e-13
    np.testing.assert_allclose(out, z["tttp"], rtol=1e-12, atol=1e-12 * np.abs(z["tttp"]).max())
    for mode in range(3):
        m = cp.mttkrp(t, factors, mode)
        assert rel(m, z[f"mttkrp{mode}"]) < 1e-13


# --------------------------------------------------------------------------
# oracle parity on BASELINE shapes

@pytest.fixture(scope="module")
def cfg2():
    shape, keys, values, factors = synth.cfg2()
    return shape, keys, values, factors


def test_cfg2_fp64_full_size_vs_oracle(cfg2):
    shape, keys, values, factors = cfg2
    t = cp.SparseTensor(shape, keys, values, validate=False)
    ot = O.OTensor(shape, keys, values)
    ref = O.tttp(ot, factors)
    got = cp.tttp(t, factors).values
    assert rel(got, ref) < 1e-12
    for mode in range(3):
        assert rel(cp.mttkrp(t, factors, mode), O.mttkrp(ot, factors, mode)) < 1e-12


def test_cfg2_fp32_residual_norm(cfg2):
    # fp32 variant: oracle = fp64 reference on fp32-rounded inputs
    torch = _torch()
    shape, keys, values, factors = cfg2
    v32 = values.astype(np.float32)
    f32 = [f.astype(np.float32) for f in factors]
    ot = O.OTensor(shape, keys, v32.astype(np.float64))
    f64r = [f.astype(np.float64) for f in f32]
    t = cp.SparseTensor(shape, keys, v32.astype(np.float64), validate=False)
    dev = [torch.from_numpy(f).cuda() for f in f32]
    got = cp.tttp(t, dev)
    assert got.device_values(torch.float32).dtype == torch.float32
    ref = O.tttp(ot, f64r)
    # residual t - model with unit mask: compare model values on the pattern
    mask = t.observation_mask()
    model = cp.tttp(mask, dev).device_values(torch.float32).double().cpu().numpy()
    omodel = O.tttp(ot.with_values(np.ones(ot.nnz)), f64r)
    r_got = np.linalg.norm(ot.values - model)
    r_ref = np.linalg.norm(ot.values - omodel)
    assert abs(r_got - r_ref) / r_ref < 1e-4
    assert rel(got.device_values(torch.float32).double().cpu().numpy(), ref) < 1e-4
    for mode in range(3):
        m = cp.mttkrp(t, dev, mode)
        assert m.dtype == torch.float32
        assert rel(m.double().cpu().numpy(), O.mttkrp(ot, f64r, mode)) < 1e-4


# --------------------------------------------------------------------------
# edge cases

def test_empty_tensor():
    t = cp.build_tensor([], (3, 3, 3))
    f = [np.ones((3, 2))] * 3
    assert np.all(cp.mttkrp(t, f, 1) == 0.0)
    assert cp.tttp(t, f) is t
    g = cp.gram_blocks(t, f, 0)
    assert g.shape == (3, 2, 2) and np.all(g == 0)
    x = cp.solve_factor(t, f, np.ones((3, 2)), 0, reg=2.0)
    assert np.allclose(x, 0.5)


@pytest.mark.parametrize("rank", [1, 2, 3, 5, 8, 10, 16, 17, 31, 32, 33, 64, 100])
def test_ranks_vs_oracle(rank):
    rng = np.random.default_rng(rank)
    dims = (37, 23, 19)
    keys = np.sort(rng.choice(np.prod(dims), 3000, replace=False)).astype(np.uint64)
    vals = rng.standard_normal(keys.size)
    fs = [rng.standard_normal((d, rank)) for d in dims]
    t = cp.SparseTensor(dims, keys, vals)
    ot = O.OTensor(dims, keys, vals)
    assert rel(cp.tttp(t, fs).values, O.tttp(ot, fs)) < 1e-13
    for mode in range(3):
        assert rel(cp.mttkrp(t, fs, mode), O.mttkrp(ot, fs, mode)) < 1e-13
    if rank <= 64:
        w = t.with_values(np.abs(vals) + 0.1)
        ow = ot.with_values(np.abs(vals) + 0.1)
        for mode in range(3):
            assert rel(cp.gram_blocks(w, fs, mode), O.gram_blocks(ow, fs, mode)) < 1e-13
            rhs = rng.standard_normal((dims[mode], rank))
            got = cp.solve_factor(w, fs, rhs, mode, reg=0.3)
            assert rel(got, O.solve_factor(ow, fs, rhs, mode, reg=0.3)) < 1e-10


@pytest.mark.parametrize("order", [2, 4, 5])
def test_orders_vs_oracle(order):
    rng = np.random.default_rng(100 + order)
    dims = tuple(int(d) for d in rng.integers(3, 12, order))
    total = int(np.prod(dims))
    keys = np.sort(rng.choice(total, min(total // 2, 4000), replace=False)).astype(np.uint64)
    vals = rng.standard_normal(keys.size)
    fs = [rng.standard_normal((d, 6)) for d in dims]
    t = cp.SparseTensor(dims, keys, vals)
    ot = O.OTensor(dims, keys, vals)
    assert rel(cp.tttp(t, fs).values, O.tttp(ot, fs)) < 1e-13
    fsn = list(fs)
    fsn[order - 1] = None
    assert rel(cp.tttp(t, fsn).values, O.tttp(ot, fsn)) < 1e-13
    for mode in range(order):
        assert rel(cp.mttkrp(t, fs, mode), O.mttkrp(ot, fs, mode)) < 1e-13
        perm, offsets = t.mode_group(mode)
        operm, ooff = ot.mode_group(mode)
        assert np.array_equal(perm, operm) and np.array_equal(offsets, ooff)


def test_skewed_rows_split_tasks():
    # a few very long rows (Zipf head) force split tasks + deterministic combine
    rng = np.random.default_rng(7)
    dims = (50, 400, 300)
    i0 = synth.zipf_indices(rng, dims[0], 60000)
    i1 = synth.zipf_indices(rng, dims[1], 60000)
    i2 = rng.integers(0, dims[2], 60000)
    t0 = cp.from_coords([i0, i1, i2], rng.integers(1, 6, 60000).astype(float), dims)
    ot = O.OTensor(dims, t0.keys, t0.values)
    fs = [rng.random((d, 32)) for d in dims]
    for task in (7, 64, 1024):
        t = cp.SparseTensor(dims, t0.keys, t0.values)
        t.set_task_size(task)
        for mode in range(3):
            a = cp.mttkrp(t, fs, mode)
            assert rel(a, O.mttkrp(ot, fs, mode)) < 1e-13
            assert np.array_equal(a, cp.mttkrp(t, fs, mode))  # run-to-run bitwise
        mask = t.observation_mask()
        omask = ot.with_values(np.ones(ot.nnz))
        for mode in range(3):
            assert rel(cp.gram_blocks(mask, fs, mode), O.gram_blocks(omask, fs, mode)) < 1e-13


def test_entry_order_invariance_bitwise():
    rng = np.random.default_rng(3)
    dims = (4, 4, 4)
    entries = [(tuple(rng.integers(0, 4, 3)), float(rng.random())) for _ in range(20)]
    t1 = cp.build_tensor(entries, dims)
    t2 = cp.build_tensor(entries[::-1], dims)
    fs = [rng.standard_normal((d, 2)) for d in dims]
    assert np.array_equal(cp.mttkrp(t1, fs, 0), cp.mttkrp(t2, fs, 0))


def test_device_resident_torch_path():
    torch = _torch()
    rng = np.random.default_rng(9)
    dims = (30, 20, 10)
    keys = np.sort(rng.choice(6000, 900, replace=False)).astype(np.uint64)
    vals = rng.standard_normal(keys.size)
    fs = [rng.standard_normal((d, 8)) for d in dims]
    t = cp.SparseTensor(dims, keys, vals)
    dfs = [torch.from_numpy(f).cuda() for f in fs]
    m = cp.mttkrp(t, dfs, 2)
    assert m.is_cuda and m.dtype == torch.float64
    assert np.array_equal(m.cpu().numpy(), cp.mttkrp(t, fs, 2))


# --------------------------------------------------------------------------
# reference known-answer tests (tests/test_kernels.py of the reference)

def test_known_answers():
    t = cp.build_tensor([((0, 0, 0), 1.0), ((0, 1, 1), 2.0)], (2, 2, 2))
    out = cp.mttkrp(t, [None, np.array([[1.0], [2.0]]), np.array([[3.0], [4.0]])], 0)
    assert out[0, 0] == 1 * 1 * 3 + 2 * 2 * 4 and out[1, 0] == 0.0
    t = cp.build_tensor([((0, 0, 0), 1.0), ((1, 1, 1), 2.0)], (2, 2, 2))
    out = cp.tttp(t, [np.array([[1.0], [2.0]]), np.array([[3.0], [4.0]]),
                      np.array([[5.0], [6.0]])])
    assert out.values.tolist() == [15.0, 96.0]
    assert np.array_equal(out.keys, t.keys)
    s = cp.build_tensor([((0, 0), 1.0), ((1, 1), 2.0)], (2, 2))
    assert cp.sddmm(s, np.array([[1.0], [2.0]]), np.array([[3.0], [4.0]])).values.tolist() \
        == [3.0, 16.0]
    w = cp.build_tensor([((0, 0, 0), 1.0)], (1, 1, 1))
    ones = [None, np.array([[1.0]]), np.array([[1.0]])]
    assert cp.solve_factor(w, ones, np.array([[5.0]]), 0, reg=0.0)[0, 0] == pytest.approx(5.0)
    assert cp.solve_factor(w, ones, np.array([[5.0]]), 0, reg=1.0)[0, 0] == pytest.approx(2.5)
    w = cp.build_tensor([((0, 0, 0), 1.0)], (3, 1, 1))
    x = cp.solve_factor(w, ones, np.array([[2.0], [4.0], [6.0]]), 0, reg=2.0)
    assert x[0, 0] == pytest.approx(2.0 / 3.0)
    assert x[1, 0] == pytest.approx(2.0) and x[2, 0] == pytest.approx(3.0)
    w = cp.build_tensor([((0, 0, 0), 1.0)], (2, 1, 1))
    x = cp.solve_factor(w, ones, np.array([[5.0], [0.0]]), 0, reg=0.0)
    assert x[1, 0] == 0.0


def test_error_semantics():
    t = cp.build_tensor([((0, 0, 0), 1.0)], (2, 2, 2))
    with pytest.raises(ValueError):
        cp.mttkrp(t, [None, None, np.ones((2, 1))], 0)
    t2 = cp.build_tensor([((0, 0), 1.0)], (2, 2))
    with pytest.raises(ValueError):
        cp.tttp(t2, [None, None])
    f = [np.random.default_rng(0).standard_normal((2, 3)) for _ in range(2)]
    with pytest.raises(ValueError):
        cp.tttp(t2, f, h_slices=0)
    with pytest.raises(ValueError):
        cp.tttp(t2, f, h_slices=4)
    with pytest.raises(ValueError):
        cp.sddmm(t, np.ones((2, 1)), np.ones((2, 1)))
    ones = [None, np.array([[1.0]]), np.array([[1.0]])]
    w = cp.build_tensor([((0, 0, 0), 1.0)], (2, 1, 1))
    with pytest.raises(cp.NumericalError, match="row 1"):
        cp.solve_factor(w, ones, np.array([[5.0], [1.0]]), 0, reg=0.0)
    w = cp.build_tensor([((0, 0, 0), -1.0)], (1, 1, 1))
    with pytest.raises(ValueError):
        cp.solve_factor(w, ones, np.array([[1.0]]), 0, reg=1.0)
    w = cp.build_tensor([((0, 0, 0), 1.0)], (1, 2, 1))
    v = np.array([[1.0], [1.0]])
    u = np.array([[1.0]])
    with pytest.raises(cp.NumericalError, match="row 0"):
        cp.solve_factor(w, [None, np.hstack([v, v]), np.hstack([u, u])],
                        np.array([[1.0, 1.0]]), 0, reg=0.0)
    with pytest.raises(ValueError):
        cp.solve_factor(w, [None, np.ones((2, 1)), np.ones((1, 1))], np.ones((1, 1)), 0,
                        reg=-1.0)


def test_gram_symmetric_psd():
    rng = np.random.default_rng(14)
    dims = (5, 5, 5)
    keys = np.flatnonzero(rng.random(125) < 0.4).astype(np.uint64)
    w = cp.SparseTensor(dims, keys, np.abs(rng.standard_normal(keys.size)))
    fs = [rng.standard_normal((d, 3)) for d in dims]
    g = cp.gram_blocks(w, fs, 0)
    for i in range(5):
        np.linalg.cholesky(g[i] + 1e-8 * np.eye(3))
        assert np.allclose(g[i], g[i].T, atol=1e-12)


@pytest.mark.parametrize("rank", [3, 16, 24, 64])
def test_fused_als_update_vs_oracle(rank):
    """cpfit_als_update: the Gram pass also accumulates the MTTKRP right-hand
    side; gram, rhs and x must match the oracle's separate mttkrp / gram /
    solve (kernels.py:46-91, 190-265), including split (Zipf-head) rows."""
    torch = _torch()
    import ctypes

    from paper_1910_02371_b200.optim import _als_mode_device
    rng = np.random.default_rng(rank)
    dims = (40, 300, 200)
    n = 40000
    i0 = synth.zipf_indices(rng, dims[0], n)
    i1 = rng.integers(0, dims[1], n)
    i2 = rng.integers(0, dims[2], n)
    t = cp.from_coords([i0, i1, i2], rng.standard_normal(n), dims)
    ot = O.OTensor(dims, t.keys, t.values)
    fs = [rng.random((d, rank)) for d in dims]
    omask = ot.with_values(np.ones(ot.nnz))
    for task in (64, 1024):
        t.set_task_size(task)
        for mode in range(3):
            F = [torch.from_numpy(f).cuda() for f in fs]
            x, gram, rhs = _als_mode_device(t, F, mode, 1e-3, keep_gram=True)
            orhs = O.mttkrp(ot, fs, mode)
            assert rel(rhs.cpu().numpy(), orhs) < 1e-12
            assert rel(gram.cpu().numpy(), O.gram_blocks(omask, fs, mode)) < 1e-12
            ox = O.solve_factor(omask, fs, orhs, mode, 1e-3)
            assert rel(x.cpu().numpy(), ox) < 1e-9
            # run-to-run bitwise
            x2 = _als_mode_device(t, F, mode, 1e-3)
            assert torch.equal(x, x2)


def test_nonfinite_factors_raise_like_reference():
    """validation.py:57-58: 'factor[n] contains non-finite entries' -- checked
    on the device after upload (cpfit_check_finite), same first error as the
    reference's host-order validation."""
    torch = _torch()
    t = cp.build_tensor([((0, 0, 0), 1.0), ((1, 1, 1), 2.0)], (2, 2, 2))
    good = np.ones((2, 3))
    bad = good.copy()
    bad[1, 2] = np.nan
    with pytest.raises(ValueError, match=r"factor\[1\] contains non-finite"):
        cp.mttkrp(t, [None, bad, good], 0)
    inf = good.copy()
    inf[0, 0] = np.inf
    with pytest.raises(ValueError, match=r"factor\[2\] contains non-finite"):
        cp.tttp(t, [good, good, inf])
    with pytest.raises(ValueError, match=r"factor\[1\] contains non-finite"):
        cp.mttkrp(t, [None, torch.from_numpy(bad).cuda(), torch.from_numpy(good).cuda()], 0)
    # first error in the reference's order: factor[0] non-finite before factor[2]'s shape
    with pytest.raises(ValueError, match=r"factor\[0\] contains non-finite"):
        cp.tttp(t, [bad, good, np.ones((3, 3))])
    with pytest.raises(ValueError, match=r"factor\[2\] has 3 rows"):
        cp.tttp(t, [good, good, np.ones((3, 3))])
    # valid calls still work after a rejected one
    assert cp.tttp(t, [good, good, good]).values.tolist() == [3.0, 6.0]


@pytest.mark.parametrize("dim1,nnz", [
    (2, 1), (2, 4095), (3, 4096), (300, 4097), (513, 8192), (1024, 12289),
    (1025, 20000), (70000, 50000), (300000, 70001), (1 << 20, 33000), ((1 << 20) + 1, 33000),
])
def test_mode_sort_digit_widths_and_tile_edges(dim1, nnz):
    """The stable LSD radix sort behind counting_sort_by_mode (core.py:234-249)
    chooses its digit width per sort and works on 4096-entry tiles: key widths of
    1 ... 21 bits (1, 2 and 3 passes, even and uneven digit splits) at entry counts
    on and next to tile edges; permutation and offsets bit-identical to numpy's
    stable argsort.  The mode-1 keys are heavily repeated (stability matters)."""
    rng = np.random.default_rng(dim1 * 7919 + nnz)
    dims = (max(2, (4 * nnz) // dim1 + 2), dim1, 5)
    total = int(np.prod([int(d) for d in dims], dtype=object))
    keys = np.unique(rng.integers(0, total, size=int(nnz * 1.3), dtype=np.int64))
    keys = np.sort(rng.choice(keys, size=min(nnz, keys.size), replace=False)).astype(np.uint64)
    t = cp.SparseTensor(dims, keys, np.ones(keys.size))
    coords = cp.delinearize_many(keys, dims)
    for mode in range(3):
        perm, offsets = t.mode_group(mode)
        want = np.argsort(coords[mode], kind="stable")
        assert np.array_equal(np.asarray(perm, dtype=np.int64), want), (mode, dims)
        counts = np.bincount(coords[mode], minlength=dims[mode])
        assert np.array_equal(np.asarray(offsets), np.concatenate(([0], np.cumsum(counts))))


def test_from_coords_wide_keys_sort():
    """Ingest sort of 60-bit linearized keys (6 passes of 10-bit digits) with
    duplicates: keys and merged values equal numpy's (core.py:208-231)."""
    rng = np.random.default_rng(3)
    dims = (1 << 20, 1 << 20, 1 << 20)
    n = 30000
    c = [rng.integers(0, d, n) for d in dims]
    for k in range(3):          # force duplicates
        c[k][n // 2:] = c[k][: n - n // 2]
    v = rng.standard_normal(n)
    t = cp.from_coords(c, v, dims)
    keys = cp.linearize_many(c, dims)
    order = np.argsort(keys, kind="stable")
    uk, start = np.unique(keys[order], return_index=True)
    assert np.array_equal(t.keys, uk)
    np.testing.assert_allclose(t.values, np.add.reduceat(v[order], start), rtol=0, atol=0)
