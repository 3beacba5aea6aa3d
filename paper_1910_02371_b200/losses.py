"""Elementwise losses, derivative tensors and fit metrics (drop-in for the
reference's losses.py).

The built-in losses (least squares and the Poisson log link, losses.py:41-91)
are evaluated on the device: model values come from the TTTP kernel on the
observation mask (losses.py:107-114), the derivative tensors from the same
kernel's loss epilogue (cpfit_tttp_loss) or the elementwise cpfit_loss_eval,
and sums from the library's fixed-order reductions; Poisson clamp events are
counted on the device and added to ``diagnostics['exp_clamped']`` exactly as
the reference's host exp() calls count them.  Losses registered by users stay
pluggable Python callables exactly as in the reference (``device_id`` None):
their elementwise phi / dphi / d2phi run on host arrays while every tensor
contraction stays on the GPU.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field
from typing import Callable

import numpy as np

from . import _lib
from .core import SparseTensor, _dtype_code, cuda_device, current_stream
from .exceptions import DataError
from .kernels import _compute_dtype, _ptrs, _to_device, tttp
from .validation import _is_torch, check_factor_list

POISSON_EXP_CLAMP = 50.0


@dataclass
class LossFunction:
    """Elementwise loss with vectorized derivative evaluators (losses.py:22-38)."""

    ident: str
    phi: Callable
    dphi: Callable
    d2phi: Callable
    validate_data: Callable = lambda values: None
    diagnostics: dict = field(default_factory=dict)
    # device evaluator of a built-in loss (csrc common.cuh loss_eval1): 0 = least
    # squares, 1 = Poisson log link; None = host callables only
    device_id: int | None = None


def least_squares() -> LossFunction:
    """phi = (t - m)^2, dphi = 2(m - t), d2phi = 2 (losses.py:41-48)."""
    return LossFunction(
        ident="ls",
        phi=lambda t, m: (t - m) ** 2,
        dphi=lambda t, m: 2.0 * (m - t),
        d2phi=lambda t, m: np.full_like(np.asarray(m, dtype=np.float64), 2.0),
        device_id=0,
    )


def poisson_log_link() -> LossFunction:
    """phi = exp(m) - t m under a clamp at m = 50 (losses.py:51-91)."""
    diagnostics = {"exp_clamped": 0}

    def _exp(m):
        m = np.asarray(m, dtype=np.float64)
        clipped = np.minimum(m, POISSON_EXP_CLAMP)
        n_clamped = int(np.count_nonzero(m > POISSON_EXP_CLAMP))
        if n_clamped:
            diagnostics["exp_clamped"] += n_clamped
        return np.exp(clipped)

    def validate_data(values):
        if np.any(np.asarray(values) < 0.0):
            raise DataError("poisson loss requires nonnegative observed values")

    return LossFunction(ident="poisson", phi=lambda t, m: _exp(m) - t * m,
                        dphi=lambda t, m: _exp(m) - t, d2phi=lambda t, m: _exp(m),
                        validate_data=validate_data, diagnostics=diagnostics, device_id=1)


_REGISTRY: dict[str, Callable[[], LossFunction]] = {
    "ls": least_squares,
    "poisson": poisson_log_link,
}


def register_loss(ident: str, factory: Callable[[], LossFunction]) -> None:
    _REGISTRY[ident] = factory


def get_loss(ident: str) -> LossFunction:
    try:
        return _REGISTRY[ident]()
    except KeyError:
        raise DataError(f"unknown loss {ident!r}; registered: {sorted(_REGISTRY)}") from None


def registered_losses() -> list[str]:
    return sorted(_REGISTRY)


# ---------------------------------------------------------------------------
# device helpers

def _reduce(op: int, x, y=None) -> float:
    out = ctypes.c_double()
    _lib.check(_lib.load().cpfit_reduce(
        op, _dtype_code(x.dtype), x.numel(), ctypes.c_void_p(x.data_ptr()),
        ctypes.c_void_p(0 if y is None else y.data_ptr()), ctypes.byref(out),
        ctypes.c_void_p(current_stream())), "reduce")
    return out.value


def sum_sq(x) -> float:
    """Deterministic sum of squares of a CUDA tensor."""
    return _reduce(0, x.contiguous())


def tttp_affine(t: SparseTensor, factors, alpha: float, beta: float, dtype=None):
    """alpha * (model at t's pattern) + beta * t.values, on the device."""
    import torch
    dtype = dtype or torch.float64
    out = torch.empty(t.nnz, dtype=dtype, device=cuda_device())
    if t.nnz == 0:
        return out
    dev = [_to_device(f, dtype) for f in factors]
    rank = next(f.shape[1] for f in dev if f is not None)
    vals = t.device_values(dtype)
    _lib.check(_lib.load().cpfit_tttp_axpby(
        t.device_pattern().handle, _dtype_code(dtype), rank, ctypes.c_void_p(vals.data_ptr()),
        _ptrs(dev), float(alpha), float(beta), ctypes.c_void_p(out.data_ptr()),
        ctypes.c_void_p(current_stream())), "tttp_axpby")
    return out


def _count_clamps(loss: LossFunction, n_clamped: int, calls: int) -> None:
    """The reference's Poisson _exp adds the clamped count once per call
    (losses.py:61-68); `calls` = how many of its exp() calls one device pass
    stands for."""
    if n_clamped and "exp_clamped" in loss.diagnostics:
        loss.diagnostics["exp_clamped"] += calls * int(n_clamped)


def device_derivatives(loss: LossFunction, t: SparseTensor, F, dtype=None):
    """(dphi, d2phi, n_clamped): device tensors at the model of factors F on
    t's pattern -- model_at_observed + derivative_tensors (losses.py:107-123)
    in one TTTP pass with the loss epilogue.  Built-in losses only; the caller
    books the clamp count (_count_clamps)."""
    import torch
    dtype = dtype or torch.float64
    d1 = torch.empty(t.nnz, dtype=dtype, device=cuda_device())
    d2 = torch.empty(t.nnz, dtype=dtype, device=cuda_device())
    if t.nnz == 0:
        return d1, d2, 0
    dev = [_to_device(f, dtype) for f in F]
    rank = next(f.shape[1] for f in dev if f is not None)
    vals = t.device_values(dtype)
    clamped = ctypes.c_int64(0)
    _lib.check(_lib.load().cpfit_tttp_loss(
        t.device_pattern().handle, _dtype_code(dtype), rank, ctypes.c_void_p(vals.data_ptr()),
        _ptrs(dev), int(loss.device_id), ctypes.c_void_p(d1.data_ptr()),
        ctypes.c_void_p(d2.data_ptr()), ctypes.byref(clamped) if loss.device_id == 1 else None,
        ctypes.c_void_p(current_stream())), "tttp_loss")
    return d1, d2, clamped.value


def _loss_eval(loss: LossFunction, tv, mv, phi=False, d1=False, d2=False):
    """Elementwise phi / dphi / d2phi of device arrays (cpfit_loss_eval)."""
    import torch
    outs = [torch.empty_like(mv) if want else None for want in (phi, d1, d2)]
    clamped = ctypes.c_int64(0)
    _lib.check(_lib.load().cpfit_loss_eval(
        int(loss.device_id), _dtype_code(mv.dtype), mv.numel(), ctypes.c_void_p(tv.data_ptr()),
        ctypes.c_void_p(mv.data_ptr()),
        *[ctypes.c_void_p(0 if o is None else o.data_ptr()) for o in outs],
        ctypes.byref(clamped) if loss.device_id == 1 else None,
        ctypes.c_void_p(current_stream())), "loss_eval")
    return outs, clamped.value


def phi_sum(loss: LossFunction, t: SparseTensor, model: SparseTensor) -> float:
    """sum phi(t, m) over the observed entries (losses.py:135)."""
    if loss.device_id is None:
        return float(np.sum(loss.phi(t.values, model.values)))
    if t.nnz == 0:
        return 0.0
    import torch
    (phi, _, _), n = _loss_eval(loss, t.device_values(torch.float64),
                                model.device_values(torch.float64), phi=True)
    _count_clamps(loss, n, 1)
    return _reduce(3, phi)


def ls_data_term(t: SparseTensor, factors, dtype=None) -> float:
    """sum (t - m)^2 over the observed entries (device)."""
    if t.nnz == 0:
        return 0.0
    return sum_sq(tttp_affine(t, factors, -1.0, 1.0, dtype))


def factor_sq_norms(factors) -> float:
    total = 0.0
    for f in factors:
        if _is_torch(f):
            total += sum_sq(f)
        else:
            total += float(np.sum(np.asarray(f) * np.asarray(f)))
    return total


# ---------------------------------------------------------------------------
# reference API

def model_at_observed(mask: SparseTensor, factors, threads: int = 1) -> SparseTensor:
    """Model values at the observed pattern = TTTP on the unit mask (losses.py:107-114)."""
    return tttp(mask, factors, threads=threads)


def derivative_tensors(loss: LossFunction, t: SparseTensor, m: SparseTensor):
    """First and second derivative tensors on the shared pattern (losses.py:117-123)."""
    if t.nnz != m.nnz or not (t._shared is m._shared or np.array_equal(t.keys, m.keys)):
        raise ValueError("observed and model tensors must share a key set")
    if loss.device_id is not None:
        import torch
        (_, d1, d2), n = _loss_eval(loss, t.device_values(torch.float64),
                                    m.device_values(torch.float64), d1=True, d2=True)
        _count_clamps(loss, n, 2)  # dphi and d2phi each call exp()
        return t.with_values(d1), t.with_values(d2)
    return (t.with_values(loss.dphi(t.values, m.values)),
            t.with_values(loss.d2phi(t.values, m.values)))


def objective(loss: LossFunction, t: SparseTensor, factors, reg: float = 0.0,
              model: SparseTensor | None = None, threads: int = 1) -> float:
    """sum phi(t, m) + reg * sum ||A_n||_F^2 (losses.py:126-138)."""
    loss.validate_data(t.values)
    if loss.ident == "ls" and model is None:
        factors_v, _ = check_factor_list(factors, t.shape)
        total = ls_data_term(t, factors_v, _compute_dtype(factors_v))
    else:
        if model is None:
            model = model_at_observed(t.observation_mask(), factors, threads=threads)
        total = phi_sum(loss, t, model)
    if reg:
        total += reg * factor_sq_norms(factors)
    return total


def rmse(t: SparseTensor, factors, model: SparseTensor | None = None,
         threads: int = 1) -> float:
    """Root-mean-square error over the observed entries (losses.py:141-150)."""
    if t.nnz == 0:
        raise ValueError("rmse undefined for an empty observation set")
    if model is None:
        factors_v, _ = check_factor_list(factors, t.shape)
        return float(np.sqrt(ls_data_term(t, factors_v, _compute_dtype(factors_v)) / t.nnz))
    import torch
    d = _reduce(1, t.device_values(torch.float64), model.device_values(torch.float64))
    return float(np.sqrt(d / t.nnz))


def fast_ls_loss(t_norm_sq: float, u_new, g_blocks, p_rhs) -> float:
    """sum t^2 + sum_i u_i^T G_i u_i - 2 sum_i u_i^T p_i (losses.py:153-171)."""
    if _is_torch(u_new) or _is_torch(g_blocks):
        import torch
        u = u_new if _is_torch(u_new) else torch.from_numpy(np.asarray(u_new)).cuda()
        g = g_blocks if _is_torch(g_blocks) else torch.from_numpy(np.asarray(g_blocks)).cuda()
        p = p_rhs if _is_torch(p_rhs) else torch.from_numpy(np.asarray(p_rhs)).cuda()
        if tuple(g.shape) != (u.shape[0], u.shape[1], u.shape[1]):
            raise ValueError("g_blocks shape does not match the updated factor")
        if tuple(p.shape) != tuple(u.shape):
            raise ValueError("p_rhs shape does not match the updated factor")
        u, g, p = u.double().contiguous(), g.double().contiguous(), p.double().contiguous()
        rank = u.shape[1]
        if rank <= 32:
            # G_i u_i by the batched symmetric mat-vec kernel, then two
            # fixed-order device dot products (no library contraction)
            gu = torch.empty_like(u)
            _lib.check(_lib.load().cpfit_batched_symv(
                _dtype_code(u.dtype), rank, u.shape[0], ctypes.c_void_p(g.data_ptr()),
                ctypes.c_void_p(u.data_ptr()), ctypes.c_void_p(gu.data_ptr()),
                ctypes.c_void_p(current_stream())), "batched_symv")
            quad = _reduce(2, u, gu)
        else:
            quad = float(torch.einsum("ir,irs,is->", u, g, u))
        cross = _reduce(2, u, p)
        return float(t_norm_sq) + quad - 2.0 * cross
    u_new = np.asarray(u_new, dtype=np.float64)
    if g_blocks.shape != (u_new.shape[0], u_new.shape[1], u_new.shape[1]):
        raise ValueError("g_blocks shape does not match the updated factor")
    if p_rhs.shape != u_new.shape:
        raise ValueError("p_rhs shape does not match the updated factor")
    quad = float(np.einsum("ir,irs,is->", u_new, g_blocks, u_new))
    cross = float(np.sum(u_new * p_rhs))
    return float(t_norm_sq) + quad - 2.0 * cross
