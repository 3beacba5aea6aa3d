"""Asynchronous result paths of the numpy API: TTTP values streaming back on
the copy stream (lazy .values), results dropped unread, interleaved calls,
non-finite factors still raising at call time, and the SM-driven pinned copy
(cpfit_copy_to_host) at odd sizes."""

import ctypes
import gc

import numpy as np
import pytest
import torch

from oracle import oracle as O

import paper_1910_02371_b200 as cp
from paper_1910_02371_b200 import _lib, synth

pytestmark = pytest.mark.gpu


def rel(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return np.linalg.norm((a - b).ravel()) / max(np.linalg.norm(b.ravel()), 1e-300)


def test_lazy_tttp_values_interleaved_and_dropped():
    shape, keys, values, factors = synth.cfg2(nnz=400_000, rank=8)
    t = cp.SparseTensor(shape, keys, values, validate=False)
    ot = O.OTensor(shape, keys, values)
    ref = O.tttp(ot, factors)
    outs = [cp.tttp(t, factors) for _ in range(3)]     # three copies in flight
    ms = [cp.mttkrp(t, factors, m) for m in range(3)]   # computed meanwhile
    for m in range(3):
        assert rel(ms[m], O.mttkrp(ot, factors, m)) < 1e-12
    for o in outs:
        assert rel(o.values, ref) < 1e-12
    for _ in range(4):  # dropped unread: the finalizer waits for the DMA
        cp.tttp(t, [f * 2.0 for f in factors])
    gc.collect()
    assert rel(cp.tttp(t, factors).values, ref) < 1e-12


def test_nonfinite_factor_still_raises_at_call():
    shape, keys, values, factors = synth.cfg2(nnz=10_000, rank=4)
    t = cp.SparseTensor(shape, keys, values, validate=False)
    bad = [f.copy() for f in factors]
    bad[1][3, 2] = np.nan
    with pytest.raises(ValueError, match=r"factor\[1\] contains non-finite entries"):
        cp.tttp(t, bad)
    with pytest.raises(ValueError, match=r"factor\[1\] contains non-finite entries"):
        cp.mttkrp(t, bad, 0)


@pytest.mark.parametrize("nbytes", [1, 15, 16, 17, 4096 + 3, 1 << 20])
def test_copy_to_host_sizes(nbytes):
    src = torch.randint(0, 255, (nbytes,), dtype=torch.uint8, device="cuda")
    dst = torch.zeros(nbytes, dtype=torch.uint8, pin_memory=True)
    _lib.check(_lib.load().cpfit_copy_to_host(
        nbytes, ctypes.c_void_p(src.data_ptr()), ctypes.c_void_p(dst.data_ptr()),
        ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)), "copy_to_host")
    torch.cuda.synchronize()
    assert torch.equal(dst, src.cpu())
    pageable = np.zeros(16, dtype=np.uint8)
    assert _lib.load().cpfit_copy_to_host(16, ctypes.c_void_p(src.data_ptr()),
                                          ctypes.c_void_p(pageable.ctypes.data), None) != 0
