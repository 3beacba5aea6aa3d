"""The reference-side binding (paper_1910_02371_b200.refbind): the reference's
numba seam (_jit.tttp3 / _jit.mttkrp3, called from kernels.py:66-74 and
:123-128) routed through the C-ABI.

* seam-level: the two drop-ins called exactly as kernels.py calls them, on a
  reference-shaped tensor (a __slots__ class like cpfit.SparseTensor,
  core.py:113), against the oracle;
* the real reference: when `cpfit` is importable (baseline/_ref, installed
  from /root/reference by pip), install the binding into it and compare its
  own kernels.mttkrp / kernels.tttp and an als_sweep with the numba path.
Needs a B200."""

import os
import sys

import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def rel(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return float(np.linalg.norm((a - b).ravel()) / max(np.linalg.norm(b.ravel()), 1e-300))


class SlotTensor:
    """Reference-shaped tensor: sorted uint64 keys + values, __slots__ like
    cpfit.SparseTensor (no attribute can be attached)."""

    __slots__ = ("shape", "keys", "values", "_coords", "_groups")

    def __init__(self, shape, keys, values):
        self.shape, self.keys, self.values = tuple(shape), keys, values
        self._coords, self._groups = None, {}

    def coords(self):
        if self._coords is None:
            self._coords = tuple(O.delinearize(self.keys, self.shape))
        return self._coords


def _case(seed=0, shape=(60, 70, 80), nnz=20000, rank=12):
    from paper_1910_02371_b200 import synth
    rng = np.random.default_rng(seed)
    keys = synth.distinct_uniform_keys(rng, int(np.prod(shape)), nnz)
    vals = rng.standard_normal(keys.size)
    fs = [rng.standard_normal((d, rank)) for d in shape]
    return shape, keys, vals, fs


def test_seam_tttp3_and_mttkrp3_vs_oracle():
    from paper_1910_02371_b200 import refbind
    shape, keys, vals, fs = _case()
    t = SlotTensor(shape, keys, vals)
    with pytest.raises(AttributeError):
        t._b200 = 1  # why the binding keeps its patterns in a side table
    ot = O.OTensor(shape, keys, vals)
    c = t.coords()
    out = np.empty(keys.size)
    refbind.tttp3(t.values, c[0], c[1], c[2], fs[0], fs[1], fs[2], out)
    assert rel(out, O.tttp(ot, fs)) < 1e-13
    refbind.tttp3(t.values * 2.0, c[0], c[1], c[2], fs[0], fs[1], fs[2], out)  # cached pattern
    assert rel(out, 2.0 * O.tttp(ot, fs)) < 1e-13
    for mode in range(3):
        # exactly kernels.py:56-74
        perm, offsets = ot.mode_group(mode)
        sorted_vals = t.values[perm]
        others = [n for n in range(3) if n != mode]
        rows_nnz = np.flatnonzero(np.diff(offsets))
        starts = offsets[rows_nnz]
        res = np.zeros((shape[mode], fs[0].shape[1]))
        refbind.mttkrp3(sorted_vals, c[others[0]][perm], c[others[1]][perm],
                        np.append(starts, offsets[-1]).astype(np.int64),
                        rows_nnz.astype(np.int64), fs[others[0]], fs[others[1]], res)
        assert rel(res, O.mttkrp(ot, fs, mode)) < 1e-13, mode


def _import_reference():
    ref = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref, "cpfit")):
        pytest.skip("reference package not installed in baseline/_ref")
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/cpfit_numba_cache")
    if ref not in sys.path:
        sys.path.insert(0, ref)
    import cpfit
    return cpfit


def test_real_reference_kernels_through_the_binding():
    cpfit = _import_reference()
    from paper_1910_02371_b200 import refbind
    shape, keys, vals, fs = _case(seed=3, shape=(200, 200, 200), nnz=80000, rank=10)
    t = cpfit.SparseTensor(shape, keys, vals)
    ref_tttp = cpfit.kernels.tttp(t, fs).values
    ref_m = [cpfit.kernels.mttkrp(t, fs, m) for m in range(3)]
    refbind.install(cpfit)
    try:
        assert cpfit._jit.tttp3 is refbind.tttp3
        got = cpfit.kernels.tttp(t, fs)
        assert np.array_equal(got.keys, t.keys)
        assert rel(got.values, ref_tttp) < 1e-13
        for m in range(3):
            assert rel(cpfit.kernels.mttkrp(t, fs, m), ref_m[m]) < 1e-13, m
    finally:
        refbind.uninstall(cpfit)
    assert cpfit._jit.tttp3 is not refbind.tttp3


def test_real_reference_als_sweep_through_the_binding():
    cpfit = _import_reference()
    from paper_1910_02371_b200 import refbind
    shape, keys, vals, _ = _case(seed=5, shape=(50, 60, 70), nnz=30000, rank=6)
    t = cpfit.SparseTensor(shape, keys, vals)
    cfg = cpfit.SolverConfig(rank=6, reg=1e-3)
    loss = cpfit.get_loss("ls")

    def sweep():
        st = cpfit.init_state(t, cfg, cpfit.RngState(7).child(0))
        for _ in range(2):
            cpfit.als_sweep(t, st, loss, cfg)
        return st.factors
    ref = sweep()
    refbind.install(cpfit)
    try:
        got = sweep()
    finally:
        refbind.uninstall(cpfit)
    for a, b in zip(got, ref):
        assert rel(a, b) < 1e-10
