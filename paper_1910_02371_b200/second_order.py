"""Second-order completion steps on the B200: Gauss-Newton / Newton with an
implicit Hessian, a block-diagonal preconditioner and PCG.

Drop-in for the reference's optim.py:334-598 (``gradient_blocks``,
``hessian_matvec``, ``BlockDiagPreconditioner``, ``pcg_solve``,
``rebalance_factors``, ``gn_step``): same signatures, validation, errors and
algorithm.  Every contraction runs on the device through the C-ABI:

* model / derivative tensors: TTTP (``cpfit_tttp_axpby``: phi1 = 2(m - t) for
  least squares; generalized losses evaluate their lambdas on the host);
* gradient: MTTKRP of phi1 plus ``2 reg A`` (``cpfit_axpby``);
* preconditioner: per-row Grams with weights phi2 (``cpfit_gram``) solved with
  ``cpfit_solve_rows`` (LU "singular" semantics of np.linalg.solve);
* Hessian matvec: ONE fused pass for z = phi2 * sum_d TTTP(A with slot d
  substituted by x_d) (``cpfit_tttp_subst``), then one MTTKRP of z per mode;
  the Newton variant adds the MTTKRPs of phi1 with one substituted slot;
* PCG on flat device vectors (one buffer holding every mode's block):
  deterministic dot products (``cpfit_reduce``) and ``cpfit_axpby`` updates;
  three host synchronisations per CG iteration (the scalars alpha, the
  residual norm and beta).
"""

from __future__ import annotations

import ctypes
import math

import numpy as np

from . import _lib
from .core import SparseTensor, _dtype_code, cuda_device, current_stream, to_host
from .exceptions import NumericalError
from .losses import LossFunction, model_at_observed, tttp_affine
from .validation import _is_torch


def _torch():
    import torch
    return torch


def _s():
    return ctypes.c_void_p(current_stream())


def _vp(t):
    return ctypes.c_void_p(0 if t is None else t.data_ptr())


def _ptrs(ts):
    return _lib.ptr_array([0 if t is None else t.data_ptr() for t in ts])


def _dev(a, dtype=None):
    torch = _torch()
    dtype = dtype or torch.float64
    if _is_torch(a):
        return a.to(device=cuda_device(), dtype=dtype).contiguous()
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).to(cuda_device()) \
        .to(dtype)


def _dot(x, y) -> float:
    out = ctypes.c_double()
    _lib.check(_lib.load().cpfit_reduce(2, _dtype_code(x.dtype), x.numel(), _vp(x), _vp(y),
                                        ctypes.byref(out), _s()), "reduce")
    return out.value


def _axpby(a, x, b, y, out):
    _lib.check(_lib.load().cpfit_axpby(_dtype_code(x.dtype), x.numel(), float(a), _vp(x),
                                       float(b), _vp(y), _vp(out), _s()), "axpby")
    return out


def _mttkrp_canon(t: SparseTensor, vals, F, mode):
    """MTTKRP with values in canonical (key) order on the device."""
    torch = _torch()
    rank = next(f for f in F if f is not None).shape[1]
    out = torch.empty((t.shape[mode], rank), dtype=vals.dtype, device=vals.device)
    ptrs = _ptrs([None if n == mode else f for n, f in enumerate(F)])
    _lib.check(_lib.load().cpfit_mttkrp(t.device_pattern().handle, mode,
                                        _dtype_code(vals.dtype), rank, _vp(vals), 0, ptrs,
                                        _vp(out), _s()), "mttkrp")
    return out


class _DeviceDerivatives:
    """phi1, phi2 (canonical order, device) of a loss at the current model."""

    def __init__(self, t: SparseTensor, F, loss: LossFunction, check_convex: bool = True):
        torch = _torch()
        self.t = t
        if t.nnz == 0:
            self.phi1 = torch.zeros(0, dtype=torch.float64, device=cuda_device())
            self.phi2 = self.phi1
            return
        if loss.ident == "ls":
            # losses.py:41-48: dphi = 2(m - t), d2phi = 2
            self.phi1 = tttp_affine(t, F, 2.0, -2.0, torch.float64)
            self.phi2 = torch.full((t.nnz,), 2.0, dtype=torch.float64, device=cuda_device())
            return
        if loss.device_id is not None:
            # built-in loss: fused TTTP loss epilogue; its d2phi (exp) is >= 0
            from .losses import _count_clamps, device_derivatives
            self.phi1, self.phi2, n = device_derivatives(loss, t, F)
            _count_clamps(loss, n, 2)
            return
        m = to_host(tttp_affine(t, F, 1.0, 0.0, torch.float64))
        p1 = np.asarray(loss.dphi(t.values, m), dtype=np.float64)
        p2 = np.asarray(loss.d2phi(t.values, m), dtype=np.float64)
        if check_convex and np.any(p2 < 0.0):
            raise NumericalError("negative second derivatives: second-order step requires a "
                                 "convex loss")
        self.phi1 = _dev(p1)
        self.phi2 = _dev(p2)


class _DeviceOperator:
    """The implicit second-order product on flat device vectors (optim.py:395-464)."""

    def __init__(self, t: SparseTensor, F, phi1, phi2, variant: str, reg: float):
        if variant not in ("gauss_newton", "newton"):
            raise ValueError(f"unknown variant {variant!r}")
        self.t, self.F, self.phi1, self.phi2 = t, F, phi1, phi2
        self.variant, self.reg = variant, float(reg)
        self.rank = F[0].shape[1]
        self.sizes = [d * self.rank for d in t.shape]
        self.offsets = np.concatenate([[0], np.cumsum(self.sizes)]).astype(np.int64)

    def blocks(self, flat):
        return [flat[self.offsets[d]:self.offsets[d + 1]].view(self.t.shape[d], self.rank)
                for d in range(self.t.order)]

    def __call__(self, pflat):
        torch = _torch()
        t, F = self.t, self.F
        x = self.blocks(pflat)
        out = torch.empty_like(pflat)
        y = self.blocks(out)
        if t.nnz:
            z = torch.empty(t.nnz, dtype=pflat.dtype, device=pflat.device)
            _lib.check(_lib.load().cpfit_tttp_subst(
                t.device_pattern().handle, _dtype_code(pflat.dtype), self.rank, _vp(self.phi2),
                _ptrs(F), _ptrs(x), _vp(z), _s()), "tttp_subst")
        for d in range(t.order):
            if t.nnz:
                m = _mttkrp_canon(t, z, F, d)
                if self.variant == "newton":
                    for p in range(t.order):
                        if p == d:
                            continue
                        sub = list(F)
                        sub[p] = x[p]
                        _axpby(1.0, _mttkrp_canon(t, self.phi1, sub, d), 1.0, m, m)
                _axpby(1.0, m, 2.0 * self.reg, x[d], y[d])
            else:
                _axpby(0.0, x[d], 2.0 * self.reg, x[d], y[d])
        return out


class _DevicePreconditioner:
    """Inverse of the per-mode diagonal blocks (G_i + shift I), optim.py:467-487.

    For rank <= 32 the blocks are inverted once, at the first application
    (``cpfit_spd_inverse_rows``), and every application is a batched
    symmetric mat-vec; a mode with a non-positive pivot keeps the pivoted
    solve per application so singular systems raise like np.linalg.solve."""

    def __init__(self, grams, shift: float, op: _DeviceOperator):
        self.grams, self.shift, self.op = grams, float(shift), op
        self.inv = None

    def _invert(self):
        torch = _torch()
        rank = self.op.rank
        self.inv = []
        for g in self.grams:
            if rank > 32 or g.shape[0] == 0:
                self.inv.append(None)
                continue
            inv = torch.empty_like(g)
            nbad = ctypes.c_int64(0)
            _lib.check(_lib.load().cpfit_spd_inverse_rows(
                _dtype_code(g.dtype), rank, g.shape[0], _vp(g), rank * rank, self.shift,
                _vp(inv), ctypes.byref(nbad), _s()), "spd_inverse_rows")
            self.inv.append(inv if nbad.value == 0 else None)

    def __call__(self, rflat):
        torch = _torch()
        if self.inv is None:
            self._invert()
        out = torch.empty_like(rflat)
        rank = self.op.rank
        for d, (r, z) in enumerate(zip(self.op.blocks(rflat), self.op.blocks(out))):
            if self.inv[d] is not None:
                _lib.check(_lib.load().cpfit_batched_symv(
                    _dtype_code(r.dtype), rank, r.shape[0], _vp(self.inv[d]), _vp(r), _vp(z),
                    _s()), "batched_symv")
                continue
            bad = ctypes.c_int64(-1)
            st = _lib.load().cpfit_solve_rows(_dtype_code(r.dtype), rank, r.shape[0],
                                              _vp(self.grams[d]), rank * rank, _vp(r),
                                              self.shift, _vp(z), ctypes.byref(bad), _s())
            if st in (_lib.ESINGULAR, _lib.EEMPTYROW):
                raise NumericalError("singular block-diagonal preconditioner; "
                                     "increase the regularization")
            _lib.check(st, "solve_rows")
        return out


def _pcg_device(matvec, precond, b, rel_tol: float, max_iters: int):
    """optim.py:492-531 on flat device vectors."""
    torch = _torch()
    if not 0.0 < rel_tol < 1.0:
        raise ValueError("rel_tol must be in (0, 1)")
    x = torch.zeros_like(b)
    r = b.clone()
    b_norm = math.sqrt(_dot(b, b))
    if b_norm == 0.0:
        return x, 0
    z = precond(r)
    p = z.clone()
    rz = _dot(r, z)
    for it in range(1, max_iters + 1):
        ap = matvec(p)
        p_ap = _dot(p, ap)
        if not math.isfinite(p_ap):
            raise NumericalError("non-finite curvature inside CG")
        if p_ap <= 0.0:
            return x, it - 1
        alpha = rz / p_ap
        _axpby(1.0, x, alpha, p, x)
        _axpby(1.0, r, -alpha, ap, r)
        res = math.sqrt(_dot(r, r))
        if not math.isfinite(res):
            raise NumericalError("non-finite residual inside CG")
        if res / b_norm < rel_tol:
            return x, it
        z = precond(r)
        rz_new = _dot(r, z)
        beta = rz_new / rz
        rz = rz_new
        _axpby(1.0, z, beta, p, p)
    return x, max_iters


def _grams(t: SparseTensor, F, phi2):
    torch = _torch()
    rank = F[0].shape[1]
    out = []
    for d in range(t.order):
        g = torch.empty((t.shape[d], rank, rank), dtype=torch.float64, device=cuda_device())
        if t.nnz:
            ptrs = _ptrs([None if n == d else f for n, f in enumerate(F)])
            st = _lib.load().cpfit_gram(t.device_pattern().handle, d, _lib.F64, rank,
                                        _vp(phi2), 0, ptrs, _vp(g), _s())
            if st == _lib.ENEGWEIGHT:
                raise ValueError("weights must be nonnegative for normal-equation assembly")
            _lib.check(st, "gram")
        else:
            g.zero_()
        out.append(g)
    return out


def _rebalance_device(F):
    """optim.py:534-555 on device factors (in place)."""
    torch = _torch()
    norms = torch.stack([torch.linalg.vector_norm(f, dim=0) for f in F])
    ok = torch.all(norms > 0.0, dim=0)
    if not bool(ok.any()):
        return
    logs = torch.log(torch.where(ok, norms, torch.ones_like(norms)))
    target = torch.exp(logs.mean(dim=0))
    for n, f in enumerate(F):
        scale = torch.where(ok, target / torch.where(ok, norms[n], torch.ones_like(norms[n])),
                            torch.ones_like(norms[n]))
        f.mul_(scale)


def gn_step_device(t: SparseTensor, F, loss: LossFunction, cfg, state, variant: str):
    """One second-order update of the device factors F (list of f64 CUDA
    tensors, updated in place); returns the CG iterations used."""
    torch = _torch()
    der = _DeviceDerivatives(t, F, loss)
    grad = [(_mttkrp_canon(t, der.phi1, F, d) if t.nnz else
             torch.zeros_like(F[d])) for d in range(t.order)]
    for d in range(t.order):
        _axpby(1.0, grad[d], 2.0 * cfg.reg, F[d], grad[d])
    grams = _grams(t, F, der.phi2)
    if cfg.gn_damping > 0.0 and state.gn_damping is None:
        diag_mean = float(np.mean([float(torch.diagonal(g, dim1=1, dim2=2).mean())
                                   for g in grams]))
        state.gn_damping = cfg.gn_damping * diag_mean
    damping = state.gn_damping or 0.0
    reg_eff = cfg.reg + damping
    op = _DeviceOperator(t, F, der.phi1, der.phi2, variant, reg_eff)
    pre = _DevicePreconditioner(grams, 2.0 * reg_eff, op)
    b = torch.cat([g.reshape(-1) for g in grad]).neg_()
    delta, used = _pcg_device(op, pre, b, cfg.cg_tol, cfg.cg_max_iters())
    for d, blk in enumerate(op.blocks(delta)):
        F[d].add_(blk)
    _rebalance_device(F)
    if state.gn_damping is not None:
        state.gn_damping *= cfg.gn_damping_decay
    return used


# ---------------------------------------------------------------------------
# reference API (numpy in / numpy out, or CUDA tensors in / out)

def _factors_dev(factors):
    return [_dev(f) for f in factors]


def _out_like(ref, dev):
    return dev if _is_torch(ref) else to_host(dev)


def gradient_blocks(t: SparseTensor, factors, loss: LossFunction, reg: float,
                    model: SparseTensor | None = None, threads: int = 1):
    """Per-mode gradient blocks: MTTKRP of the dphi tensor plus 2 reg A
    (optim.py:336-345)."""
    F = _factors_dev(factors)
    if model is not None and loss.device_id is not None and t.nnz:
        from .losses import _count_clamps, _loss_eval
        (_, phi1, _), n = _loss_eval(loss, t.device_values(_torch().float64),
                                     model.device_values(_torch().float64), d1=True)
        _count_clamps(loss, n, 1)
    elif model is not None:
        p1 = np.asarray(loss.dphi(t.values, model.values), dtype=np.float64)
        phi1 = _dev(p1)
    else:
        phi1 = _DeviceDerivatives(t, F, loss, check_convex=False).phi1
    out = []
    for d in range(t.order):
        g = _mttkrp_canon(t, phi1, F, d) if t.nnz else _torch().zeros_like(F[d])
        _axpby(1.0, g, 2.0 * reg, F[d], g)
        out.append(_out_like(factors[d], g))
    return out


def hessian_matvec(phi1: SparseTensor, phi2: SparseTensor, factors, x_blocks,
                   variant: str = "gauss_newton", reg: float = 0.0, threads: int = 1):
    """Implicit second-order product (optim.py:348-384): z = phi2 * sum_d
    TTTP(A with slot d -> x_d), y_d = MTTKRP(z, d) + 2 reg x_d (+ the Newton
    cross terms MTTKRP(phi1, A with one slot p != d -> x_p, d))."""
    if variant not in ("gauss_newton", "newton"):
        raise ValueError(f"unknown variant {variant!r}")
    n_modes = len(factors)
    if len(x_blocks) != n_modes:
        raise ValueError("one update block per mode required")
    for d in range(n_modes):
        if tuple(x_blocks[d].shape) != tuple(factors[d].shape):
            raise ValueError(f"update block {d} shape mismatch")
    F = _factors_dev(factors)
    f64 = _torch().float64
    op = _DeviceOperator(phi2, F, phi1.device_values(f64), phi2.device_values(f64), variant,
                         reg)
    flat = _torch().cat([_dev(x).reshape(-1) for x in x_blocks])
    y = op(flat)
    return [_out_like(x_blocks[d], blk.contiguous()) for d, blk in enumerate(op.blocks(y))]


class BlockDiagPreconditioner:
    """Inverse of the per-mode diagonal blocks of the second-order model
    (optim.py:467-487): (G_i + reg I) per row, G from ``gram_blocks`` with
    phi2 weights, applied with the batched device solve."""

    def __init__(self, phi2: SparseTensor, factors, reg: float, row_batches: int = 1,
                 threads: int = 1, grams=None):
        self.reg = float(reg)
        self.rank = factors[0].shape[1]
        if grams is not None:
            self.grams = [_dev(g) for g in grams]
        else:
            F = _factors_dev(factors)
            self.grams = _grams(phi2, F, phi2.device_values(_torch().float64))

    def apply(self, blocks):
        out = []
        for g, b in zip(self.grams, blocks):
            rhs = _dev(b)
            z = _torch().empty_like(rhs)
            bad = ctypes.c_int64(-1)
            st = _lib.load().cpfit_solve_rows(_lib.F64, self.rank, rhs.shape[0], _vp(g),
                                              self.rank * self.rank, _vp(rhs), self.reg,
                                              _vp(z), ctypes.byref(bad), _s())
            if st in (_lib.ESINGULAR, _lib.EEMPTYROW):
                raise NumericalError("singular block-diagonal preconditioner; "
                                     "increase the regularization")
            _lib.check(st, "solve_rows")
            out.append(_out_like(b, z))
        return out


def _block_dot(a, b) -> float:
    total = 0.0
    for x, y in zip(a, b):
        if _is_torch(x):
            total += _dot(x.contiguous().reshape(-1), y.contiguous().reshape(-1))
        else:
            total += float(np.sum(x * y))
    return total


def pcg_solve(matvec, precond, rhs_blocks, rel_tol: float, max_iters: int):
    """Preconditioned conjugate gradient over lists of factor-shaped blocks
    (optim.py:492-531; numpy or CUDA-tensor blocks)."""
    if not 0.0 < rel_tol < 1.0:
        raise ValueError("rel_tol must be in (0, 1)")
    x = [_torch().zeros_like(b) if _is_torch(b) else np.zeros_like(b) for b in rhs_blocks]
    r = [b.copy() if not _is_torch(b) else b.clone() for b in rhs_blocks]
    b_norm = math.sqrt(_block_dot(rhs_blocks, rhs_blocks))
    if b_norm == 0.0:
        return x, 0
    z = precond(r)
    p = [zi.copy() if not _is_torch(zi) else zi.clone() for zi in z]
    rz = _block_dot(r, z)
    for it in range(1, max_iters + 1):
        ap = matvec(p)
        p_ap = _block_dot(p, ap)
        if not math.isfinite(p_ap):
            raise NumericalError("non-finite curvature inside CG")
        if p_ap <= 0.0:
            return x, it - 1
        alpha = rz / p_ap
        for d in range(len(x)):
            x[d] = x[d] + alpha * p[d]
            r[d] = r[d] - alpha * ap[d]
        res = math.sqrt(_block_dot(r, r))
        if not math.isfinite(res):
            raise NumericalError("non-finite residual inside CG")
        if res / b_norm < rel_tol:
            return x, it
        z = precond(r)
        rz_new = _block_dot(r, z)
        beta = rz_new / rz
        rz = rz_new
        for d in range(len(p)):
            p[d] = z[d] + beta * p[d]
    return x, max_iters


def rebalance_factors(factors) -> None:
    """Equalize each component's column norms across modes, in place
    (optim.py:534-555)."""
    if all(_is_torch(f) for f in factors):
        _rebalance_device(factors)
        return
    norms = np.stack([np.linalg.norm(f, axis=0) for f in factors])
    ok = np.all(norms > 0.0, axis=0)
    if not np.any(ok):
        return
    target = np.exp(np.log(norms[:, ok]).mean(axis=0))
    for n in range(len(factors)):
        scale = np.ones(norms.shape[1])
        scale[ok] = target / norms[n, ok]
        factors[n] *= scale


def gn_step(t: SparseTensor, state, loss: LossFunction, cfg,
            variant: str = "gauss_newton") -> int:
    """One second-order update of all factors at once (optim.py:558-598)."""
    host = not any(_is_torch(f) for f in state.factors)
    F = _factors_dev(state.factors)
    used = gn_step_device(t, F, loss, cfg, state, variant)
    if host:
        state.factors = [to_host(f).copy() for f in F]
    else:
        state.factors = F
    return used


__all__ = ["gradient_blocks", "hessian_matvec", "BlockDiagPreconditioner", "pcg_solve",
           "rebalance_factors", "gn_step", "gn_step_device", "model_at_observed"]
