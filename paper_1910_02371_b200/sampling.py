"""Device Bernoulli sampling of a tensor's entries (SparseTensor.sample).

Keeps entry e iff draw e of ``RngState.generator().random(nnz)`` is < rate,
exactly as the reference (core.py:173-183): the device kernel regenerates
numpy's Philox4x64-10 stream bit for bit (draw e = word e % 4 of
philox(counter=[e//4 + 1, 0, 0, 0], key)), then compacts survivors in order.
The sample is born on the device (coordinates gathered into a new pattern,
values gathered); host keys/values materialise only if asked for.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib
from .core import (DevicePattern, SparseTensor, _Shared, _dtype_code, current_stream,
                   device_view)


def sample_pattern(t: SparseTensor, rate: float, rng, counter_offset: int = 0):
    """Return (DevicePattern of survivors, int32 CUDA tensor of parent positions)."""
    if not 0.0 < rate <= 1.0:
        raise ValueError(f"sample rate must be in (0, 1], got {rate}")
    k0, k1 = rng.philox_key()
    out = ctypes.c_void_p()
    src = t.device_pattern()
    _lib.check(_lib.load().cpfit_sample(src.handle, k0, k1, int(counter_offset), float(rate),
                                        ctypes.c_void_p(current_stream()), ctypes.byref(out)),
               "sample")
    n = ctypes.c_int64()
    _lib.check(_lib.load().cpfit_pattern_info(out, None, ctypes.byref(n)))
    pat = DevicePattern(t.shape, n.value, out.value)
    if t._shared.task_size is not None:
        _lib.check(_lib.load().cpfit_pattern_set_task_size(pat.handle, t._shared.task_size))
    idx = ctypes.c_void_p()
    _lib.check(_lib.load().cpfit_pattern_parent_index(pat.handle, ctypes.byref(idx)))
    parent = device_view(idx.value, n.value, "<i4", pat)
    return pat, parent


def gather_values(values, parent):
    """values[parent] on the device (library kernel)."""
    import torch
    out = torch.empty(parent.numel(), dtype=values.dtype, device=values.device)
    _lib.check(_lib.load().cpfit_gather_values(
        _dtype_code(values.dtype), parent.numel(), ctypes.c_void_p(parent.data_ptr()),
        ctypes.c_void_p(values.data_ptr()), ctypes.c_void_p(out.data_ptr()),
        ctypes.c_void_p(current_stream())), "gather_values")
    return out


def sample_tensor(t: SparseTensor, rate: float, rng, dtype=None,
                  counter_offset: int = 0) -> SparseTensor:
    """Bernoulli sample of t's entries; entry e uses Philox draw
    counter_offset + e (a nonzero shard passes its first global index)."""
    if not 0.0 < rate <= 1.0:
        raise ValueError(f"sample rate must be in (0, 1], got {rate}")
    import torch
    dtype = dtype or torch.float64
    if t.nnz == 0:
        return SparseTensor(t.shape, np.empty(0, np.uint64), np.empty(0), validate=False)
    pat, parent = sample_pattern(t, rate, rng, counter_offset)
    vals = gather_values(t.device_values(dtype), parent)
    shared = _Shared(pattern=pat, task_size=t._shared.task_size, parent=parent)
    host_parent = {}

    def keys_fn():
        if "p" not in host_parent:
            host_parent["p"] = parent.cpu().numpy()
        return t.keys[host_parent["p"]]

    return SparseTensor._device_born(t.shape, pat.nnz, shared, vals, keys_fn=keys_fn)
