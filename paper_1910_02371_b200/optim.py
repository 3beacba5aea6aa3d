"""Completion drivers on the B200: ALS, CCD++ and SGD sweeps and ``run``.

Drop-in for the reference's optim.py (SolverConfig / CompletionState /
init_state / als_sweep / ccd_sweep / sgd_sweep / run, same semantics,
validation and messages).  With the least-squares loss every sweep runs on
the device end to end:

* ALS (optim.py:180-207): per mode, MTTKRP of the data (rhs) and the fused
  Gram assembly + batched SPD solve with unit weights (the observation mask is
  never materialised); reg, not 2 reg, on the diagonal.
* CCD++ (optim.py:235-268): the residual lives on the device as rhat (the
  residual with column r added back, every mode's rho); each (r, mode) step
  is one segmented num/den pass, and rhat is re-formed once per column.
* SGD (optim.py:300-330): bit-exact device Philox sample, derivative tensor
  2(m - t) fused into TTTP, sampled MTTKRPs at the pre-step factors, update
  in numpy's evaluation order.

Factor matrices may be numpy arrays (results written back as numpy, like the
reference) or CUDA tensors (kept on the device).  Generalized losses follow
the reference's inner-Newton formulation using the same kernels.
"""

from __future__ import annotations

import ctypes
import math
import time
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .core import RngState, SparseTensor, _dtype_code, cuda_device, current_stream
from .exceptions import NumericalError
from .kernels import _ptrs, gram_blocks, mttkrp, solve_factor, tttp
from .losses import (LossFunction, derivative_tensors, factor_sq_norms, get_loss,
                     ls_data_term, model_at_observed, phi_sum, tttp_affine)
from .second_order import (BlockDiagPreconditioner, gn_step, gradient_blocks,  # noqa: F401
                           hessian_matvec, pcg_solve, rebalance_factors)
from .trace import RunTrace
from .validation import _is_torch

ALGORITHMS = ("als", "ccd", "sgd", "gn", "newton")
_INIT_LAWS = ("uniform", "gaussian", "svd")
_TINY = 1e-300


@dataclass
class SolverConfig:
    """Settings for a completion run (optim.py:30-89)."""

    rank: int = 10
    algorithm: str = "als"
    loss: str = "ls"
    reg: float = 1e-5
    max_iters: int = 20
    tol: float = 1e-6
    inner_max: int = 5
    inner_tol: float = 1e-3
    cg_tol: float = 5e-3
    cg_max: int | None = None
    step: float = 5e-3
    sample_rate: float = 1.0
    init: str = "uniform"
    seed: int = 0
    deterministic: bool = False
    threads: int = 1
    row_batches: int = 1
    h_slices: int | None = None
    record_every: int | None = None
    freeze_curvature: bool = False
    calibrate_init: bool = False
    gn_damping: float = 0.0
    gn_damping_decay: float = 0.5
    warmup_sweeps: int = 0
    # not in the reference: "direct" = its per-row LAPACK solve (batched
    # Cholesky here); "cg" = Gram-free per-row conjugate gradients (BASELINE
    # cfg 3 "ALS completion with implicit CG"), stopped by cg_tol / cg_max
    als_solver: str = "direct"

    def __post_init__(self):
        # the reference's rules and messages (optim.py:62-86), as a table: the
        # first failing row raises
        positive = [n for n in ("tol", "inner_tol", "cg_tol", "step") if getattr(self, n) <= 0]
        rules = (
            (self.rank >= 1, "rank must be >= 1"),
            (self.algorithm in ALGORITHMS, f"unknown algorithm {self.algorithm!r}"),
            (self.reg >= 0, "reg must be >= 0"),
            (self.max_iters >= 0, "max_iters must be >= 0"),
            (not positive, f"{positive[0] if positive else ''} must be positive"),
            (0.0 < self.sample_rate <= 1.0, "sample_rate must be in (0, 1]"),
            (self.cg_tol < 1.0, "cg_tol must be in (0, 1)"),
            (self.init in _INIT_LAWS, f"unknown init law {self.init!r}"),
            (min(self.threads, self.inner_max, self.row_batches) >= 1,
             "threads, inner_max, row_batches must be >= 1"),
            (self.gn_damping >= 0 and 0.0 < self.gn_damping_decay <= 1.0,
             "gn_damping must be >= 0 and its decay in (0, 1]"),
            (self.warmup_sweeps >= 0, "warmup_sweeps must be >= 0"),
            (self.als_solver in ("direct", "cg"), f"unknown als_solver {self.als_solver!r}"),
        )
        for ok, message in rules:
            if not ok:
                raise ValueError(message)

    def cg_max_iters(self) -> int:
        return self.cg_max if self.cg_max is not None else min(30, 3 * self.rank)


@dataclass
class CompletionState:
    """Mutable solver state: the factor matrices plus per-sweep caches."""

    factors: list
    rng: RngState
    iteration: int = 0
    ls_gram: list = field(default_factory=list)
    ls_rhs: list = field(default_factory=list)
    gn_damping: float | None = None

    def __post_init__(self):
        if not self.ls_gram:
            self.ls_gram = [None] * len(self.factors)
        if not self.ls_rhs:
            self.ls_rhs = [None] * len(self.factors)


def init_state(t: SparseTensor, cfg: SolverConfig, rng: RngState | None = None
               ) -> CompletionState:
    """Initial factors (host draws in the reference's order, optim.py:113-146:
    one (I_n x R) block per mode from ``RngState(seed).child(0)``, scaled by
    1/sqrt(R)); uploaded by the drivers, never regenerated on the device."""
    rng = rng or RngState(cfg.seed).child(0)
    g = rng.generator()
    scale = 1.0 / math.sqrt(cfg.rank)
    draw = {"uniform": g.random, "gaussian": g.standard_normal}
    factors = [
        draw[cfg.init]((extent, cfg.rank)) * scale if cfg.init in draw
        else _svd_init_factor(t, mode, cfg.rank, g, scale)
        for mode, extent in enumerate(t.shape)
    ]
    if cfg.calibrate_init and t.nnz:
        _calibrate_scale(t, factors)
    return CompletionState(factors=factors, rng=rng)


def _calibrate_scale(t: SparseTensor, factors) -> None:
    """Least-squares scalar c = <t, m> / <m, m> between the data and the initial
    model m, spread evenly over the modes (|c|^(1/N) each, the sign on mode 0);
    optim.py:131-145."""
    model = tttp(t.observation_mask(), factors).values
    mm = float(np.dot(model, model))
    if mm <= 0.0:
        return
    c = float(np.dot(t.values, model)) / mm
    if c == 0.0:
        return
    per_mode = abs(c) ** (1.0 / t.order)
    for f in factors:
        f *= per_mode
    if c < 0.0:
        factors[0] *= -1.0


def _svd_init_factor(t, mode, rank, g, scale):
    """Leading left singular vectors of the mode-``mode`` unfolding (scipy
    ``svds`` on the host, as optim.py:149-174; initialisation only).  Columns
    the unfolding cannot supply are uniform draws."""
    from scipy.sparse import csr_matrix
    from scipy.sparse.linalg import svds
    coords = t.coords()
    n_rows = t.shape[mode]
    others = [n for n in range(t.order) if n != mode]
    n_cols = math.prod(t.shape[n] for n in others)
    k = min(rank, n_rows - 1, n_cols - 1)
    if k < 1:
        return g.random((n_rows, rank)) * scale
    cols = np.zeros(t.nnz, dtype=np.int64)
    for n in others:                       # column = row-major key of the other modes
        cols = cols * t.shape[n] + coords[n]
    unfolding = csr_matrix((t.values, (coords[mode], cols)), shape=(n_rows, n_cols))
    u = svds(unfolding, k=k, return_singular_vectors="u",
             random_state=np.random.RandomState(0))[0]
    out = np.empty((n_rows, rank))
    out[:, :k] = u[:, ::-1]                # svds returns ascending singular values
    if k < rank:
        out[:, k:] = g.random((n_rows, rank - k)) * scale
    return np.ascontiguousarray(out)


# ---------------------------------------------------------------------------
# device factor handling

def _torch():
    import torch
    return torch


def _to_dev_factors(factors, dtype=None):
    torch = _torch()
    out = []
    for f in factors:
        if _is_torch(f):
            out.append(f.to(cuda_device()).contiguous() if dtype is None
                       else f.to(device=cuda_device(), dtype=dtype).contiguous())
        else:
            out.append(torch.from_numpy(np.ascontiguousarray(f, dtype=np.float64))
                       .to(cuda_device()).to(dtype or torch.float64))
    return out


def _write_back(state_factors, dev):
    for n, f in enumerate(state_factors):
        if _is_torch(f):
            state_factors[n] = dev[n]
        else:
            state_factors[n] = dev[n].double().cpu().numpy()


def _stream():
    return ctypes.c_void_p(current_stream())


# ---------------------------------------------------------------------------
# alternating minimization

def _als_mode_device(t: SparseTensor, F, mode: int, reg: float, keep_gram: bool = False,
                     row_offset: int = 0):
    """One least-squares ALS mode update on the device: the Gram assembly
    with the MTTKRP right-hand side fused in (unit weights: the observation
    mask is never materialised) + batched SPD solve.  Returns x (or (x, gram, rhs))
    with t.shape[mode] rows; F[mode] is not read (t's mode may be a rebased
    row block of a larger factor -- dist.ShardedALS)."""
    torch = _torch()
    dtype = F[0].dtype if F[0] is not None else F[1].dtype
    dev = next(f for f in F if f is not None).device
    code = _dtype_code(dtype)
    rank = next(f for f in F if f is not None).shape[1]
    L = _lib.load()
    pat = t.device_pattern()
    ptrs = _ptrs([None if n == mode else f for n, f in enumerate(F)])
    rhs = torch.empty((t.shape[mode], rank), dtype=dtype, device=dev)
    vals = t.sorted_values(mode, dtype) if t.nnz else None
    x = torch.empty_like(rhs)
    # always a torch-cached buffer: a library-side scratch of I_n x R x R would
    # hit the stream-ordered pool's allocate/release path on every call
    gram = torch.empty((t.shape[mode], rank, rank), dtype=dtype, device=dev)
    bad = ctypes.c_int64(-1)
    # rhs (MTTKRP of the data) accumulated by the Gram pass itself: one gather
    # of the factor rows per entry (cpfit_als_update)
    st = L.cpfit_als_update(pat.handle, mode, code, rank,
                            None if vals is None else ctypes.c_void_p(vals.data_ptr()), 1, ptrs,
                            float(reg), ctypes.c_void_p(x.data_ptr()),
                            ctypes.c_void_p(gram.data_ptr()), ctypes.c_void_p(rhs.data_ptr()),
                            ctypes.byref(bad), _stream())
    if st == _lib.EEMPTYROW:
        raise NumericalError(
            f"alternating solve failed: mode {mode} row {bad.value + row_offset}: no incident "
            "entries and reg=0 but right-hand side is nonzero")
    if st == _lib.ESINGULAR:
        raise NumericalError(f"alternating solve failed: mode {mode} row "
                             f"{bad.value + row_offset}: singular normal equations "
                             f"(reg={float(reg)})")
    _lib.check(st, "als_update")
    if keep_gram:
        return x, gram, rhs
    return x


def _als_mode_cg_device(t: SparseTensor, F, mode: int, reg: float, tol: float, max_iters: int,
                        warm_start: bool = True, weights=None, rhs=None):
    """One least-squares ALS mode update without Gram blocks ("ALS completion
    with implicit CG", BASELINE cfg 3): rhs = MTTKRP of the data, then every
    row's (G_i + reg I) x_i = rhs_i by conjugate gradients whose product G_i p_i
    is one pass over the nonzeros (cpfit_gram_matvec); rows carry their own
    alpha / beta and drop out of the passes as they converge (pcg_solve's
    stopping rule, optim.py:521-523, per row).  Warm-started from F[mode].
    Returns (x, rhs, iterations).  Peak extra memory: five I_n x R arrays
    instead of the I_n x R x R Gram buffer."""
    torch = _torch()
    ref = next(f for n, f in enumerate(F) if f is not None and n != mode)
    dtype, dev, rank = ref.dtype, ref.device, ref.shape[1]
    code = _dtype_code(dtype)
    L = _lib.load()
    pat = t.device_pattern()
    rows = t.shape[mode]
    ptrs = _ptrs([None if n == mode else f for n, f in enumerate(F)])
    st = _stream()
    if rhs is None:
        rhs = torch.empty((rows, rank), dtype=dtype, device=dev)
        vals = t.sorted_values(mode, dtype) if t.nnz else None
        _lib.check(L.cpfit_mttkrp(pat.handle, mode, code, rank,
                                  None if vals is None else ctypes.c_void_p(vals.data_ptr()), 1,
                                  ptrs, ctypes.c_void_p(rhs.data_ptr()), st), "mttkrp")
    wptr = None if weights is None else ctypes.c_void_p(weights.data_ptr())

    def matvec(v, active, out):
        _lib.check(L.cpfit_gram_matvec(pat.handle, mode, code, rank, wptr, 1, ptrs,
                                       ctypes.c_void_p(v.data_ptr()),
                                       None if active is None else ctypes.c_void_p(active.data_ptr()),
                                       ctypes.c_void_p(out.data_ptr()), st), "gram_matvec")

    q = torch.empty_like(rhs)
    r = torch.empty_like(rhs)
    p = torch.empty_like(rhs)
    rho = torch.empty(rows, dtype=torch.float64, device=dev)
    thresh2 = torch.empty(rows, dtype=torch.float64, device=dev)
    active = torch.empty(rows, dtype=torch.int32, device=dev)
    status = torch.zeros(2, dtype=torch.int64, device=dev)
    if warm_start and F[mode] is not None:
        x = F[mode].to(dtype).clone()
        matvec(x, None, q)
        ax = ctypes.c_void_p(q.data_ptr())
    else:
        x = torch.zeros_like(rhs)
        ax = None
    vp = lambda a: ctypes.c_void_p(a.data_ptr())  # noqa: E731
    _lib.check(L.cpfit_cg_rows_init(code, rows, rank, float(reg), float(tol), vp(rhs), ax, vp(x),
                                    vp(r), vp(p), vp(rho), vp(thresh2), vp(active), vp(status),
                                    st), "cg_rows_init")
    iters = 0
    live, bad = status.tolist()
    while live and not bad and iters < max_iters:
        matvec(p, active, q)
        _lib.check(L.cpfit_cg_rows_step(code, rows, rank, float(reg), vp(q), vp(x), vp(r), vp(p),
                                        vp(rho), vp(thresh2), vp(active), vp(status), st),
                   "cg_rows_step")
        iters += 1
        live, bad = status.tolist()
    if bad:
        raise NumericalError("non-finite curvature inside CG")
    return x, rhs, iters


def _als_ls_cg_device(t: SparseTensor, F, reg: float, tol: float, max_iters: int):
    """One implicit-CG least-squares ALS sweep on device factors (modes in
    order, optim.py:194-206).  Returns per-mode (rhs, CG iterations)."""
    rhss, iters = [], []
    for mode in range(t.order):
        x, rhs, it = _als_mode_cg_device(t, F, mode, reg, tol, max_iters)
        F[mode] = x
        rhss.append(rhs)
        iters.append(it)
    return rhss, iters


def _als_ls_device(t: SparseTensor, F, reg: float, keep_gram: bool = True):
    """One least-squares ALS sweep on device factors F (list of CUDA tensors,
    updated in place, modes in order, optim.py:194-206).  Returns per-mode
    (gram, rhs)."""
    grams, rhss = [], []
    for mode in range(t.order):
        if keep_gram:
            x, gram, rhs = _als_mode_device(t, F, mode, reg, keep_gram=True)
        else:
            x, gram, rhs = _als_mode_device(t, F, mode, reg), None, None
        F[mode] = x
        grams.append(gram)
        rhss.append(rhs)
    return grams, rhss


def als_sweep(t: SparseTensor, state: CompletionState, loss: LossFunction,
              cfg: SolverConfig, generalized: bool | None = None) -> None:
    """One pass of alternating minimization over all modes, in order
    (optim.py:180-229)."""
    if generalized is None:
        generalized = loss.ident != "ls"
    if not generalized and cfg.als_solver == "cg":
        F = _to_dev_factors(state.factors)
        rhss, _ = _als_ls_cg_device(t, F, cfg.reg, cfg.cg_tol, cfg.cg_max_iters())
        host = not any(_is_torch(f) for f in state.factors)
        for mode in range(t.order):
            state.ls_gram[mode] = None  # never formed
            state.ls_rhs[mode] = rhss[mode].cpu().numpy() if host else rhss[mode]
        _write_back(state.factors, F)
        return
    if not generalized:
        F = _to_dev_factors(state.factors)
        grams, rhss = _als_ls_device(t, F, cfg.reg)
        host = not any(_is_torch(f) for f in state.factors)
        for mode in range(t.order):
            state.ls_gram[mode] = grams[mode].cpu().numpy() if host else grams[mode]
            state.ls_rhs[mode] = rhss[mode].cpu().numpy() if host else rhss[mode]
        _write_back(state.factors, F)
        return
    if loss.device_id is not None:
        F = _to_dev_factors(state.factors)
        _als_generalized_device(t, F, loss, cfg)
        _write_back(state.factors, F)
        return
    mask = t.observation_mask()
    for mode in range(t.order):
        phi2 = None
        for inner in range(cfg.inner_max):
            model = model_at_observed(mask, state.factors, threads=cfg.threads)
            phi1, phi2_new = derivative_tensors(loss, t, model)
            if phi2 is None or not cfg.freeze_curvature:
                phi2 = phi2_new
            grad = _as_np(mttkrp(phi1, state.factors, mode))
            grad = grad + 2.0 * cfg.reg * _as_np(state.factors[mode])
            try:
                delta = _as_np(solve_factor(phi2, state.factors, -grad, mode,
                                            reg=2.0 * cfg.reg, row_batches=cfg.row_batches))
            except NumericalError as err:
                raise NumericalError(f"inner Newton solve failed: {err}") from err
            new = _as_np(state.factors[mode]) + delta
            state.factors[mode] = _like(state.factors[mode], new)
            rel = np.linalg.norm(delta) / max(np.linalg.norm(new), _TINY)
            if rel < cfg.inner_tol:
                break


def _axpby(a: float, x, b: float, y, out):
    _lib.check(_lib.load().cpfit_axpby(_dtype_code(x.dtype), x.numel(), float(a),
                                       ctypes.c_void_p(x.data_ptr()), float(b),
                                       ctypes.c_void_p(y.data_ptr()),
                                       ctypes.c_void_p(out.data_ptr()), _stream()), "axpby")
    return out


def _als_generalized_device(t: SparseTensor, F, loss: LossFunction, cfg: SolverConfig):
    """Inner-Newton alternating sweep of a built-in loss on device factors
    (optim.py:208-229): per mode and inner step, the derivative tensors at the
    current model in one fused TTTP pass (cpfit_tttp_loss), the gradient
    MTTKRP(dphi) + 2 reg A, the phi2-weighted Gram + batched solve with 2 reg
    on the diagonal, and the update; the inner stopping test reads two
    fixed-order device norms."""
    from .losses import _count_clamps, device_derivatives, sum_sq
    torch = _torch()
    for mode in range(t.order):
        phi2 = None
        for inner in range(cfg.inner_max):
            d1, d2, n = device_derivatives(loss, t, F)
            _count_clamps(loss, n, 2)
            if phi2 is None or not cfg.freeze_curvature:
                phi2 = t.with_values(d2)
            grad = mttkrp(t.with_values(d1), F, mode)
            _axpby(1.0, grad, 2.0 * cfg.reg, F[mode], grad)  # grad += 2 reg A (numpy order)
            _axpby(-1.0, grad, 0.0, grad, grad)
            try:
                delta = solve_factor(phi2, F, grad, mode, reg=2.0 * cfg.reg,
                                     row_batches=cfg.row_batches)
            except NumericalError as err:
                raise NumericalError(f"inner Newton solve failed: {err}") from err
            new = torch.empty_like(F[mode])
            F[mode] = _axpby(1.0, F[mode], 1.0, delta, new)
            rel = math.sqrt(sum_sq(delta)) / max(math.sqrt(sum_sq(new)), _TINY)
            if rel < cfg.inner_tol:
                break


def _as_np(a):
    return a.double().cpu().numpy() if _is_torch(a) else np.asarray(a, dtype=np.float64)


def _like(ref, a):
    if _is_torch(ref):
        return _torch().from_numpy(a).to(ref.device).to(ref.dtype)
    return a


# ---------------------------------------------------------------------------
# coordinate minimization

def _ccd_col_ptrs(cols, r=None):
    """Pointer array to column r of every mode (cols[n] is R x I_n), or to the
    vectors themselves when r is None."""
    arr = _lib.ptr_array([(c if r is None else c[r]).data_ptr() for c in cols])
    return arr, ctypes.cast(arr, ctypes.POINTER(ctypes.c_void_p))


def _ccd_rhat_copies(t: SparseTensor, resid, lean: bool):
    """rhat copies: mode n's in its mode-sorted order (mode 0: canonical), or
    the canonical one only (lean: modes > 0 read it through the permutation)."""
    torch = _torch()
    if lean:
        return [resid]
    copies = [resid]
    for n in range(1, t.order):
        out = torch.empty_like(resid)
        if t.nnz:
            _lib.check(_lib.load().cpfit_permute_values(
                t.device_pattern().handle, n, _dtype_code(torch.float64),
                ctypes.c_void_p(resid.data_ptr()), ctypes.c_void_p(out.data_ptr()),
                _stream()), "permute_values")
        copies.append(out)
    return copies


def _ccd_lean(t: SparseTensor) -> bool:
    """One canonical rhat when the per-mode copies would not fit comfortably."""
    torch = _torch()
    need = (t.order - 1) * t.nnz * 8
    try:
        free, _ = torch.cuda.mem_get_info()
    except RuntimeError:
        return False
    return need > free // 2


def _ccd_ls_device(t: SparseTensor, F, reg: float, lean: bool | None = None):
    """CCD++ least-squares sweep on device factors (list of f64 CUDA tensors).

    Column r keeps rhat = resid + (rank-one term of column r) on the device:
    it is every mode's rho of the reference (optim.py:254) in exact
    arithmetic, so each (r, mode) update is one segmented (num, den) pass.
    Every mode holds its own copy of rhat in its mode-sorted order and
    re-forms it for column r inside its own pass (csrc/ccd.cu).  Returns the
    residual t - model."""
    torch = _torch()
    order = t.order
    rank = F[0].shape[1]
    L = _lib.load()
    pat = t.device_pattern()
    if lean is None:
        lean = _ccd_lean(t)
    cols = [f.t().contiguous() for f in F]  # R x I_n: column r contiguous
    resid = tttp_affine(t, F, -1.0, 1.0, torch.float64)  # t - model
    rh = _ccd_rhat_copies(t, resid, lean)
    old = [torch.empty(d, dtype=torch.float64, device=resid.device) for d in t.shape]
    old_keep, old_ptrs = _ccd_col_ptrs(old)
    prev = None
    for r in range(rank):
        keep, ptrs = _ccd_col_ptrs(cols, r)
        sub = prev[1] if prev is not None else None
        if lean:
            # canonical copy only: re-formed in the mode-0 pass (identity order,
            # column r untouched there, so cols themselves are the "old" values)
            for mode in range(order):
                f = mode == 0
                _lib.check(L.cpfit_ccd_step(
                    pat.handle, mode, ptrs, ctypes.c_void_p(rh[0].data_ptr()), 0,
                    sub if f else None, ptrs if f else None, float(reg), None, _stream()),
                    "ccd_step")
        else:
            for n in range(order):
                old[n].copy_(cols[n][r])
            for mode in range(order):
                _lib.check(L.cpfit_ccd_step(
                    pat.handle, mode, ptrs, ctypes.c_void_p(rh[mode].data_ptr()), 1, sub,
                    old_ptrs, float(reg), None, _stream()), "ccd_step")
        prev = (keep, ptrs)
    if prev is not None:
        _lib.check(L.cpfit_ccd_fold(pat.handle, -1, prev[1], None,
                                    ctypes.c_void_p(rh[0].data_ptr()), _stream()), "ccd_fold")
    for n in range(order):
        F[n] = cols[n].t().contiguous()
    return rh[0]


def ccd_sweep(t: SparseTensor, state: CompletionState, loss: LossFunction,
              cfg: SolverConfig) -> None:
    """One coordinate-minimization sweep, column-then-mode order (optim.py:235-294)."""
    if loss.ident == "ls":
        F = _to_dev_factors(state.factors, _torch().float64)
        _ccd_ls_device(t, F, cfg.reg)
        _write_back(state.factors, F)
        return
    # built-in losses evaluate dphi / d2phi on the device; a user-registered
    # loss runs the same device sweep with its host callables
    F = _to_dev_factors(state.factors, _torch().float64)
    _ccd_generalized_device(t, F, loss, cfg)
    _write_back(state.factors, F)


def _ccd_generalized_device(t: SparseTensor, F, loss: LossFunction, cfg: SolverConfig):
    """Inner-Newton CCD++ sweep of a built-in loss on device factors
    (optim.py:269-294): per (r, mode, inner step) the weights part * dphi and
    part^2 * d2phi at the current model (cpfit_ccd_gen_weights; for a
    user-registered loss its dphi / d2phi callables run on the model values
    copied to the host, as the reference evaluates them), their row
    sums (two R = 1 MTTKRPs against unit columns), the damped-free Newton
    column update and the model update; the stopping test reads two
    fixed-order device norms."""
    from .losses import _count_clamps, sum_sq, tttp_affine
    torch = _torch()
    L = _lib.load()
    order = t.order
    rank = F[0].shape[1]
    dev = F[0].device
    f64 = torch.float64
    pat = t.device_pattern()
    cols = [f.t().contiguous() for f in F]  # R x I_n
    if t.nnz:
        model = tttp_affine(t.observation_mask(), F, 1.0, 0.0, f64)
    else:
        model = torch.zeros(0, dtype=f64, device=dev)
    tv = t.device_values(f64)
    w1 = torch.empty_like(model)
    w2 = torch.empty_like(model)
    part = torch.empty_like(model)
    ones = [torch.ones((d, 1), dtype=f64, device=dev) for d in t.shape]
    ones_ptrs = _ptrs(ones)
    deltas = [torch.empty(d, dtype=f64, device=dev) for d in t.shape]
    clamped = ctypes.c_int64(0)
    count = loss.device_id == 1
    user = loss.device_id is None
    lid = 2 if user else int(loss.device_id)
    t_host = t.values if user else None
    for r in range(rank):
        keep, ptrs = _ccd_col_ptrs(cols, r)
        for mode in range(order):
            col = cols[mode][r]
            num = torch.zeros((t.shape[mode], 1), dtype=f64, device=dev)
            den = torch.zeros((t.shape[mode], 1), dtype=f64, device=dev)
            for inner in range(cfg.inner_max):
                if t.nnz:
                    a1, a2 = tv, model
                    if user:
                        m_host = model.cpu().numpy()
                        a1 = torch.from_numpy(np.ascontiguousarray(
                            loss.dphi(t_host, m_host), dtype=np.float64)).to(dev)
                        a2 = torch.from_numpy(np.ascontiguousarray(
                            loss.d2phi(t_host, m_host), dtype=np.float64)).to(dev)
                    _lib.check(L.cpfit_ccd_gen_weights(
                        pat.handle, mode, lid, ptrs,
                        ctypes.c_void_p(a1.data_ptr()), ctypes.c_void_p(a2.data_ptr()),
                        ctypes.c_void_p(w1.data_ptr()), ctypes.c_void_p(w2.data_ptr()),
                        ctypes.c_void_p(part.data_ptr()),
                        ctypes.byref(clamped) if count else None, _stream()), "ccd_gen_weights")
                    if count:
                        _count_clamps(loss, clamped.value, 2)  # dphi and d2phi
                    for w, out in ((w1, num), (w2, den)):
                        _lib.check(L.cpfit_mttkrp(pat.handle, mode, _dtype_code(f64), 1,
                                                  ctypes.c_void_p(w.data_ptr()), 0, ones_ptrs,
                                                  ctypes.c_void_p(out.data_ptr()), _stream()),
                                   "mttkrp")
                delta = deltas[mode]
                _lib.check(L.cpfit_ccd_gen_update(
                    t.shape[mode], ctypes.c_void_p(num.data_ptr()),
                    ctypes.c_void_p(den.data_ptr()), float(cfg.reg),
                    ctypes.c_void_p(col.data_ptr()), ctypes.c_void_p(delta.data_ptr()),
                    _stream()), "ccd_gen_update")
                if t.nnz:
                    _lib.check(L.cpfit_ccd_gen_model(
                        pat.handle, mode, ctypes.c_void_p(part.data_ptr()),
                        ctypes.c_void_p(delta.data_ptr()), ctypes.c_void_p(model.data_ptr()),
                        _stream()), "ccd_gen_model")
                rel = math.sqrt(sum_sq(delta)) / max(math.sqrt(sum_sq(col)), _TINY)
                if rel < cfg.inner_tol:
                    break
    for n in range(order):
        F[n] = cols[n].t().contiguous()


# ---------------------------------------------------------------------------
# stochastic gradient descent

def _sgd_grads_device(t: SparseTensor, F, rate: float, rng: RngState, dtype,
                      counter_offset: int = 0, loss: LossFunction | None = None):
    """Sample (global Philox counter starts at counter_offset) and the per-mode
    gradients MTTKRP(dphi) on the device -- least squares 2(m - t) through the
    TTTP affine epilogue, other built-in losses through its loss epilogue;
    returns (grads, sample nnz)."""
    torch = _torch()
    from .sampling import sample_tensor
    code = _dtype_code(dtype)
    L = _lib.load()
    sampled = sample_tensor(t, rate, rng, dtype, counter_offset=counter_offset)
    rank = F[0].shape[1]
    if sampled.nnz == 0:
        return [torch.zeros((t.shape[m], rank), dtype=dtype, device=F[0].device)
                for m in range(t.order)], 0
    if loss is None or loss.device_id == 0:
        phi1 = tttp_affine(sampled, F, 2.0, -2.0, dtype)  # 2(m - t), losses.py:46
    elif loss.device_id is None:
        # user-registered loss: model on the device, its host dphi on the values
        model = tttp_affine(sampled, F, 1.0, 0.0, torch.float64).cpu().numpy()
        d1 = np.ascontiguousarray(loss.dphi(sampled.values, model), dtype=np.float64)
        phi1 = torch.from_numpy(d1).to(device=F[0].device, dtype=dtype)
    else:
        from .losses import _count_clamps, device_derivatives
        phi1, _, n = device_derivatives(loss, sampled, F, dtype)
        _count_clamps(loss, n, 1)  # sgd_sweep evaluates dphi only (optim.py:320)
    pat = sampled.device_pattern()
    grads = []
    for mode in range(t.order):
        g = torch.empty((t.shape[mode], rank), dtype=dtype, device=F[0].device)
        _lib.check(L.cpfit_mttkrp(pat.handle, mode, code, rank,
                                  ctypes.c_void_p(phi1.data_ptr()), 0, _ptrs(F),
                                  ctypes.c_void_p(g.data_ptr()), _stream()), "mttkrp")
        grads.append(g)
    return grads, sampled.nnz


def _sgd_apply_device(F, grads, step: float, shrink: float, check: bool = True):
    """F[n] <- (F[n] - step*grad_n) - shrink*F[n] for every mode at once."""
    torch = _torch()
    L = _lib.load()
    new = []
    for mode, f in enumerate(F):
        out = torch.empty_like(f)
        bad = ctypes.c_int(0)
        _lib.check(L.cpfit_sgd_update(_dtype_code(f.dtype), f.numel(), ctypes.c_void_p(f.data_ptr()),
                                      ctypes.c_void_p(grads[mode].data_ptr()), float(step),
                                      float(shrink), ctypes.c_void_p(out.data_ptr()),
                                      ctypes.byref(bad), _stream()), "sgd_update")
        if bad.value and check:
            raise NumericalError(f"sgd update diverged on mode {mode}; the learning rate is "
                                 "too high for this sample rate")
        new.append(out)
    for mode in range(len(F)):
        F[mode] = new[mode]


def _sgd_ls_device(t: SparseTensor, F, cfg: SolverConfig, rng: RngState,
                   loss: LossFunction | None = None):
    """One SGD step on device factors F (list of CUDA tensors, replaced);
    least squares unless a built-in `loss` is given."""
    shrink = 2.0 * cfg.step * cfg.reg * cfg.sample_rate
    grads, n = _sgd_grads_device(t, F, cfg.sample_rate, rng, F[0].dtype, loss=loss)
    _sgd_apply_device(F, grads, cfg.step, shrink, check=n > 0)
    return n


def sgd_sweep(t: SparseTensor, state: CompletionState, loss: LossFunction,
              cfg: SolverConfig, rng: RngState) -> None:
    """One sampled gradient step on all factors at once (optim.py:300-330)."""
    dtype = None
    if all(_is_torch(f) and f.dtype == _torch().float32 for f in state.factors):
        dtype = _torch().float32
    F = _to_dev_factors(state.factors, dtype)
    _sgd_ls_device(t, F, cfg, rng, loss)
    _write_back(state.factors, F)


# ---------------------------------------------------------------------------
# orchestration

def _one_iteration(t, state, loss, cfg, it: int, sgd_rng: RngState) -> None:
    """One outer iteration of the configured algorithm (optim.py:655-664)."""
    algo = cfg.algorithm
    if algo == "sgd":
        sgd_sweep(t, state, loss, cfg, sgd_rng.child(it))   # fresh sample stream per step
    elif algo in ("gn", "newton"):
        gn_step(t, state, loss, cfg, variant="gauss_newton" if algo == "gn" else "newton")
    else:
        {"als": als_sweep, "ccd": ccd_sweep}[algo](t, state, loss, cfg)
    state.iteration = it


def _require_finite_factors(factors, it: int) -> None:
    # a NaN / inf anywhere in a factor makes its sum non-finite: one reduction
    # per factor on whichever side (device or host) it lives
    for d, f in enumerate(factors):
        total = float(f.sum()) if _is_torch(f) else float(np.sum(f))
        if not np.isfinite(total):
            raise NumericalError(f"factor {d} became non-finite at iteration {it}; "
                                 "reduce the step size or increase reg")


def run(t: SparseTensor, cfg: SolverConfig, return_state: bool = False):
    """Run the configured solver and collect a convergence trace.

    Same contract as the reference's ``run`` (optim.py:604-691): record 0 is the
    initial point; a record every ``record_every`` iterations (default 20 for
    SGD, else 1) and at the last one; stop when the relative objective change
    between records drops below ``tol``; NumericalError on non-finite factors
    or a diverged objective.  Built-in losses keep the factors on the device
    for the whole run and evaluate the objective there."""
    loss = get_loss(cfg.loss)
    loss.validate_data(t.values)
    root = RngState(cfg.seed)
    state = init_state(t, cfg, root.child(0))
    sgd_rng = root.child(1)
    every = cfg.record_every if cfg.record_every is not None else (
        20 if cfg.algorithm == "sgd" else 1)
    is_ls = loss.ident == "ls"
    trace = RunTrace(
        metric_name="rmse" if is_ls else "norm_loss",
        metadata={"algorithm": cfg.algorithm, "loss": cfg.loss, "rank": str(cfg.rank),
                  "reg": repr(cfg.reg), "seed": str(cfg.seed),
                  "shape": "x".join(map(str, t.shape)), "nnz": str(t.nnz)},
    )
    on_device = loss.device_id is not None
    if on_device:
        state.factors = _to_dev_factors(state.factors)
    mask = t.observation_mask()
    count = max(t.nnz, 1)
    t_start = time.perf_counter()

    def seconds() -> float:
        if cfg.deterministic:       # byte-stable traces
            return 0.0
        _torch().cuda.synchronize()
        return time.perf_counter() - t_start

    def evaluate():
        """(objective, metric): data term + reg * ||factors||^2, and rmse (least
        squares) or the mean loss."""
        if is_ls:
            data = ls_data_term(t, state.factors)
            metric = float(np.sqrt(data / count))
        else:
            data = phi_sum(loss, t, model_at_observed(mask, state.factors, threads=cfg.threads))
            metric = data / count
        return data + cfg.reg * factor_sq_norms(state.factors), metric

    if cfg.algorithm in ("gn", "newton"):
        for _ in range(cfg.warmup_sweeps):
            als_sweep(t, state, loss, cfg)
    obj, metric = evaluate()
    trace.append(0, seconds(), obj, metric)
    first_obj = last_obj = obj
    for it in range(1, cfg.max_iters + 1):
        _one_iteration(t, state, loss, cfg, it, sgd_rng)
        _require_finite_factors(state.factors, it)
        if it % every and it != cfg.max_iters:
            continue
        obj, metric = evaluate()
        trace.append(it, seconds(), obj, metric)
        if not math.isfinite(obj) or obj > 1e3 * max(abs(first_obj), 1.0):
            raise NumericalError(f"objective diverged at iteration {it}: {obj!r} from "
                                 f"{first_obj!r}; reduce the step size or increase reg")
        if abs(last_obj - obj) / max(abs(last_obj), _TINY) < cfg.tol:
            break
        last_obj = obj
    if on_device:
        state.factors = [f.double().cpu().numpy() for f in state.factors]
    return (trace, state) if return_state else trace
