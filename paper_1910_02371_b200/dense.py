"""Dense-tensor MTTKRP and CP-ALS (BASELINE cfg 4: 800^3 fp64, R = 64).

The reference has no dense tensor type; its oracle for this row
is ``kernels.mttkrp`` / ``als_sweep`` on a fully observed SparseTensor
(kernels.py:46-91, optim.py:180-207), against which tests/test_gpu_dense.py
checks these functions.

Every contraction runs in this library's own kernels (no cuBLAS):

* ``dense_mttkrp(X, F, mode)`` -- einsum('ijk,jr,kr->ir') and its mode-1 /
  mode-2 analogues as ONE pass over X with the Khatri-Rao operand formed in
  shared memory (``cpfit_dense_mttkrp``): FP64 DMMA for float64 (the parity
  path), TF32 ``tcgen05.mma`` with TMEM accumulators for float32.
* ``dense_als_sweep`` -- one CP-ALS sweep.  Modes 0 and 1 share
  T = X_(IJ x K) C (``cpfit_dense_xc``, same kernel family; C does not change
  between them) reduced by ``cpfit_dense_reduce``; mode 2 is one KR pass with
  the updated A and B.  Two passes over X per sweep instead of three.  The
  per-mode normal equations share one Gram, the Hadamard product of the
  other factors' R x R Gramians (``cpfit_dense_gram``; every entry of a dense
  tensor is observed), solved for all rows by ``cpfit_solve_rows`` (reg on
  the diagonal, like ``solve_factor``).
"""

from __future__ import annotations

import ctypes

from . import _lib
from .core import _dtype_code, current_stream
from .exceptions import NumericalError


def _torch():
    import torch
    return torch


def _s():
    return ctypes.c_void_p(current_stream())


def _vp(t):
    return ctypes.c_void_p(t.data_ptr() if t is not None else 0)


def _check_dense(X, factors):
    torch = _torch()
    if X.dim() != 3:
        raise ValueError("dense_mttkrp supports order-3 tensors")
    if not X.is_cuda:
        raise ValueError("dense tensors must be CUDA tensors")
    if X.dtype not in (torch.float64, torch.float32):
        raise ValueError(f"unsupported dtype {X.dtype}")
    if len(factors) != 3:
        raise ValueError("dense_mttkrp needs three factor slots")
    rank = None
    for n, f in enumerate(factors):
        if f is None:
            continue
        if f.dim() != 2 or f.shape[0] != X.shape[n]:
            raise ValueError(f"factor {n} must have shape ({X.shape[n]}, R)")
        if rank is not None and f.shape[1] != rank:
            raise ValueError("factor ranks disagree")
        rank = f.shape[1]
    if rank is None:
        raise ValueError("at least one factor is required")
    return rank


def _prep(f, dtype):
    return None if f is None else f.to(dtype).contiguous()


def dense_mttkrp(X, factors, mode: int):
    """einsum('ijk,jr,kr->ir') (mode 0) and its mode-1 / mode-2 analogues for
    an order-3 dense CUDA tensor X (float64: FP64 tensor cores; float32:
    TF32 tcgen05).  The factor in slot ``mode`` is ignored (may be None)."""
    torch = _torch()
    rank = _check_dense(X, factors)
    if mode not in (0, 1, 2):
        raise ValueError(f"mode {mode} out of range for order-3 tensor")
    X = X.contiguous()
    A, B, C = (_prep(f, X.dtype) for f in factors)
    needed = {0: (B, C), 1: (A, C), 2: (A, B)}[mode]
    if any(f is None for f in needed):
        raise ValueError(f"mode {mode} needs the other two factors")
    I, J, K = X.shape
    out = torch.empty((X.shape[mode], rank), dtype=X.dtype, device=X.device)
    _lib.check(_lib.load().cpfit_dense_mttkrp(_dtype_code(X.dtype), I, J, K, rank, _vp(X),
                                              _vp(A), _vp(B), _vp(C), mode, _vp(out), _s()),
               "dense_mttkrp")
    return out


def xc_product(X, C):
    """T[i, j, :] = X[i, j, :] @ C   (the GEMM shared by modes 0 and 1)."""
    torch = _torch()
    I, J, K = X.shape
    C = C.to(X.dtype).contiguous()
    T = torch.empty((I, J, C.shape[1]), dtype=X.dtype, device=X.device)
    _lib.check(_lib.load().cpfit_dense_xc(_dtype_code(X.dtype), I, J, K, C.shape[1],
                                          _vp(X.contiguous()), _vp(C), _vp(T), _s()),
               "dense_xc")
    return T


def reduce_t(T, W, axis: int):
    torch = _torch()
    I, J, R = T.shape
    out = torch.empty((I if axis == 1 else J, R), dtype=T.dtype, device=T.device)
    _lib.check(_lib.load().cpfit_dense_reduce(_dtype_code(T.dtype), I, J, R, _vp(T),
                                              _vp(W.contiguous()), axis, _vp(out), _s()),
               "dense_reduce")
    return out


def khatri_rao(A, B):
    torch = _torch()
    I, R = A.shape
    J = B.shape[0]
    out = torch.empty((I * J, R), dtype=A.dtype, device=A.device)
    _lib.check(_lib.load().cpfit_khatri_rao(_dtype_code(A.dtype), I, J, R, _vp(A.contiguous()),
                                            _vp(B.contiguous()), _vp(out), _s()), "khatri_rao")
    return out


def gram_hadamard(factors):
    """G = prod_f F_f^T F_f (elementwise), R x R, on the device."""
    torch = _torch()
    fs = [f.contiguous() for f in factors]
    rank = fs[0].shape[1]
    G = torch.empty((rank, rank), dtype=fs[0].dtype, device=fs[0].device)
    rows = (ctypes.c_int64 * len(fs))(*[f.shape[0] for f in fs])
    _lib.check(_lib.load().cpfit_dense_gram(_dtype_code(fs[0].dtype), len(fs), rows, rank,
                                            _lib.ptr_array([f.data_ptr() for f in fs]),
                                            _vp(G), _s()), "dense_gram")
    return G


def solve_shared(G, rhs, reg: float):
    """x_i = (G + reg I)^-1 rhs_i for every row i (one shared SPD G)."""
    torch = _torch()
    rank = G.shape[0]
    x = torch.empty_like(rhs)
    bad = ctypes.c_int64(-1)
    st = _lib.load().cpfit_solve_rows(_dtype_code(rhs.dtype), rank, rhs.shape[0],
                                      _vp(G.contiguous()), 0, _vp(rhs.contiguous()), float(reg),
                                      _vp(x), ctypes.byref(bad), _s())
    if st == _lib.ESINGULAR:
        raise NumericalError(f"singular normal equations (reg={float(reg)})")
    _lib.check(st, "solve_rows")
    return x


def dense_als_sweep(X, factors, reg: float):
    """One CP-ALS sweep (modes in order, reg on the diagonal as in the
    reference's least-squares als_sweep, optim.py:192-206); factors are CUDA
    tensors, replaced in the list."""
    _check_dense(X, factors)
    X = X.contiguous()
    T = xc_product(X, factors[2])  # C is unchanged while modes 0 and 1 update
    for mode in range(3):
        others = [factors[n] for n in range(3) if n != mode]
        G = gram_hadamard(others)
        if mode == 0:
            M = reduce_t(T, factors[1], axis=1)
        elif mode == 1:
            M = reduce_t(T, factors[0], axis=0)
        else:
            M = dense_mttkrp(X, factors, 2)
        factors[mode] = solve_shared(G, M, reg)
    return factors


__all__ = ["dense_mttkrp", "dense_als_sweep", "gram_hadamard", "khatri_rao", "solve_shared",
           "xc_product"]
