"""Reference-side binding: route the reference package's compiled seam through
this library's C-ABI.

The reference (`cpfit`) has exactly one compiled seam, the numba kernels in
its ``_jit`` module, which ``kernels.mttkrp`` / ``kernels.tttp`` call when
``t.order == 3 and _jit.HAS_NUMBA`` (kernels.py:66-74 and :123-128):

    _jit.tttp3(vals, i0, i1, i2, f0, f1, f2, out)            # out[e] = v_e sum_r a b c
    _jit.mttkrp3(sorted_vals, idx_a, idx_b, starts, rows,     # out[rows[g]] +=
                 fac_a, fac_b, out)                           #   sum (a b) v over group g

``install(cpfit)`` replaces those two functions (and ``set_threads``) with
the ones below, so every caller -- kernels.mttkrp/tttp, hence als_sweep,
sgd_sweep, gn_step, rmse, ... -- runs the sm_100a kernels with the reference's
own validation, caching and drivers around them.  ``uninstall`` restores the
originals.

Device patterns are cached in a side table, because ``cpfit.SparseTensor``
uses ``__slots__`` (core.py:113) and cannot carry an attribute:

* TTTP receives the tensor's cached coordinate arrays (``t.coords()``, shared
  by every ``with_values`` copy), so the pattern is keyed by the identity of
  the mode-0 coordinate array and dropped when that array is collected;
* MTTKRP receives freshly permuted arrays (kernels.py:60-62) already in the
  target mode's stable order, i.e. canonical order for the mode permutation
  (target, a, b); a pattern over those three coordinate
  arrays is built per call and MTTKRP runs on its mode 0.

This is the binding INTEGRATION.md describes; tests/test_gpu_refbind.py runs it
against the real reference when it is importable (baseline/_ref).
"""

from __future__ import annotations

import ctypes
import weakref

import numpy as np

from . import _lib
from .core import DevicePattern, current_stream, cuda_device

_F64 = 0
_PATTERNS: dict = {}   # id(mode-0 coords array) -> DevicePattern
_SAVED: dict = {}      # id(module) -> original seam functions


def _torch():
    import torch
    return torch


def _dev_i32(a):
    torch = _torch()
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.int32)).to(cuda_device())


def _dev_f64(a):
    torch = _torch()
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).to(cuda_device())


def _pattern_from(coords) -> DevicePattern:
    """Pattern over per-mode coordinates in canonical order; dims = max + 1
    (the seam does not pass the shape; TTTP / mode-0 MTTKRP do not need it)."""
    dims = tuple(int(c.max()) + 1 if c.size else 1 for c in coords)
    return DevicePattern.from_device_coords(dims, [_dev_i32(c) for c in coords])


def _tttp_pattern(i0, i1, i2) -> DevicePattern:
    key = id(i0)
    hit = _PATTERNS.get(key)
    if hit is not None and hit[1]() is i0:
        return hit[0]
    pat = _pattern_from([i0, i1, i2])
    try:
        ref = weakref.ref(i0, lambda _r, k=key: _PATTERNS.pop(k, None))
    except TypeError:  # not weak-referenceable: no caching
        return pat
    _PATTERNS[key] = (pat, ref)
    return pat


def tttp3(vals, i0, i1, i2, f0, f1, f2, out) -> None:
    """Drop-in for _jit.tttp3 (_jit.py:49-59): out[e] = vals[e] * sum_r
    f0[i0[e], r] f1[i1[e], r] f2[i2[e], r], written into the caller's array."""
    n = int(np.asarray(vals).shape[0])
    if n == 0:
        return
    torch = _torch()
    pat = _tttp_pattern(i0, i1, i2)
    fs = [_dev_f64(f) for f in (f0, f1, f2)]
    v = _dev_f64(vals)
    res = torch.empty(n, dtype=torch.float64, device=cuda_device())
    arr = _lib.ptr_array([f.data_ptr() for f in fs])
    _lib.check(_lib.load().cpfit_tttp(pat.handle, _F64, int(fs[0].shape[1]),
                                      ctypes.c_void_p(v.data_ptr()), arr,
                                      ctypes.c_void_p(res.data_ptr()),
                                      ctypes.c_void_p(current_stream())), "tttp")
    out[:] = res.cpu().numpy()


def mttkrp3(sorted_vals, idx_a, idx_b, starts, rows, fac_a, fac_b, out) -> None:
    """Drop-in for _jit.mttkrp3 (_jit.py:35-47): for each group g, out[rows[g]]
    += sum over sorted positions starts[g]:starts[g+1] of (a * b) * v."""
    n = int(np.asarray(sorted_vals).shape[0])
    if n == 0 or len(rows) == 0:
        return
    torch = _torch()
    starts = np.asarray(starts, dtype=np.int64)
    rows = np.asarray(rows, dtype=np.int64)
    target = np.repeat(rows, np.diff(starts))          # entry -> output row
    pat = _pattern_from([target, idx_a, idx_b])         # canonical for (target, a, b)
    rank = int(np.asarray(fac_a).shape[1])
    fa, fb = _dev_f64(fac_a), _dev_f64(fac_b)
    v = _dev_f64(sorted_vals)
    dim0 = pat.shape[0]
    res = torch.empty((dim0, rank), dtype=torch.float64, device=cuda_device())
    arr = _lib.ptr_array([0, fa.data_ptr(), fb.data_ptr()])
    _lib.check(_lib.load().cpfit_mttkrp(pat.handle, 0, _F64, rank,
                                        ctypes.c_void_p(v.data_ptr()), 1, arr,
                                        ctypes.c_void_p(res.data_ptr()),
                                        ctypes.c_void_p(current_stream())), "mttkrp")
    out[rows] += res.cpu().numpy()[rows]


def set_threads(threads: int) -> None:
    """The device path is independent of the host thread count."""


def install(cpfit) -> None:
    """Route ``cpfit``'s numba seam (``cpfit._jit``) to the sm_100a kernels."""
    jit = cpfit._jit
    if id(jit) not in _SAVED:
        _SAVED[id(jit)] = (jit, {name: getattr(jit, name, None)
                                 for name in ("HAS_NUMBA", "tttp3", "mttkrp3", "set_threads")})
    jit.tttp3 = tttp3
    jit.mttkrp3 = mttkrp3
    jit.set_threads = set_threads
    jit.HAS_NUMBA = True  # take the order-3 seam branch in kernels.py


def uninstall(cpfit) -> None:
    """Restore the reference's own seam functions."""
    jit = cpfit._jit
    saved = _SAVED.pop(id(jit), None)
    if saved is None:
        return
    for name, fn in saved[1].items():
        if fn is None:
            if hasattr(jit, name):
                delattr(jit, name)
        else:
            setattr(jit, name, fn)


__all__ = ["install", "uninstall", "tttp3", "mttkrp3", "set_threads"]
