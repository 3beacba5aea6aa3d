"""All-at-once multi-tensor kernels on the B200: MTTKRP, TTTP/SDDMM, Gram and
factor solves.

Drop-in for the reference's kernels.py (same signatures, validation, error
types and messages).  Each function validates on the host, then calls one
hand-written sm_100a kernel of ``libcpfit_b200.so`` through the C-ABI
(include/cpfit_b200.h) on the current torch CUDA stream.  There is no CPU
fallback.

Inputs: factor matrices may be numpy arrays (the reference's API: they are
uploaded, results come back as numpy) or CUDA ``torch.Tensor`` (device
resident; results stay on the device as tensors).  float32 CUDA factors select
the fp32 kernels; everything else computes in float64 like the reference.

Results are deterministic run to run (no floating-point atomics); ``threads``
is accepted for signature compatibility and ignored, as the reference's
results are thread-count independent too (kernels.py:12-15).
"""

from __future__ import annotations

import os

import ctypes

import numpy as np

from . import _lib
from .core import SparseTensor, _dtype_code, cuda_device, current_stream, to_host, to_host_sm
from .exceptions import NumericalError
from .validation import _is_torch, check_factor, check_factor_list, check_mode

DEFAULT_TTTP_BUDGET_BYTES = 1 << 28
DEFAULT_STAGE_ROWS = 256


def _torch():
    import torch
    return torch


def _compute_dtype(arrays):
    """float32 only when every provided operand is a float32 CUDA tensor."""
    torch = _torch()
    provided = [a for a in arrays if a is not None]
    if provided and all(_is_torch(a) and a.dtype == torch.float32 for a in provided):
        return torch.float32
    return torch.float64


def _device_mode(arrays) -> bool:
    return any(_is_torch(a) for a in arrays if a is not None)


def _to_device(a, dtype):
    torch = _torch()
    if a is None:
        return None
    if _is_torch(a):
        return a.to(device=cuda_device(), dtype=dtype).contiguous()
    # non_blocking: pinned sources copy asynchronously; pageable ones are
    # staged by the driver before the call returns (safe to reuse either way)
    return torch.from_numpy(np.ascontiguousarray(a)).to(cuda_device(), non_blocking=True) \
        .to(dtype)


def _checked_factor_list(factors, dims, **kw):
    """check_factor_list with the non-finite scan deferred to the device.
    On a host-side (shape / rank) error the full host validation re-runs so
    the first error raised is the reference's (validation.py:62-95 order)."""
    try:
        return check_factor_list(factors, dims, finite=False, **kw)
    except ValueError:
        check_factor_list(factors, dims, finite=True, **kw)
        raise


class _FiniteCheck:
    """Deferred 'contains non-finite entries' check (validation.py:57-58):
    one cpfit_check_finite launch per uploaded operand into a device flag
    array; ``raise_if_bad`` reads the flags after the call's own result
    synchronisation and raises the reference's ValueError for the first bad
    operand (the computed result is discarded)."""

    def __init__(self, named):
        torch = _torch()
        self.named = [(n, d) for n, d in named if d is not None and d.numel()]
        self.flags = None
        if not self.named:
            return
        self.flags = torch.zeros(len(self.named), dtype=torch.int32, device=cuda_device())
        L = _lib.load()
        base = self.flags.data_ptr()
        for k, (_, d) in enumerate(self.named):
            _lib.check(L.cpfit_check_finite(_dtype_code(d.dtype), d.numel(), _vp(d),
                                            ctypes.c_void_p(base + 4 * k), _stream()),
                       "check_finite")
        # flags head to the host right behind the checks (written by a kernel
        # into pinned memory: a copy-engine transfer would queue behind any
        # large device->host copy still draining), so reading them waits for
        # the checks only
        self.host = torch.empty(len(self.named), dtype=torch.int32, pin_memory=True)
        _lib.check(L.cpfit_copy_to_host(4 * len(self.named), ctypes.c_void_p(base),
                                        ctypes.c_void_p(self.host.data_ptr()), _stream()),
                   "copy_to_host")
        self.done = torch.cuda.Event()
        self.done.record()

    def raise_if_bad(self):
        if self.flags is None:
            return
        self.done.synchronize()
        bad = self.host.numpy()
        for k, (name, _) in enumerate(self.named):
            if bad[k]:
                raise ValueError(f"{name} contains non-finite entries")


def _named(factors, dev):
    return [(f"factor[{n}]", d) for n, d in enumerate(dev) if factors[n] is not None]


def _ptrs(tensors):
    return _lib.ptr_array([0 if t is None else t.data_ptr() for t in tensors])


def _vp(t):
    return ctypes.c_void_p(0 if t is None else t.data_ptr())


def _stream():
    return ctypes.c_void_p(current_stream())


# ---------------------------------------------------------------------------

_MTTKRP_DIRECT_HOST = os.environ.get("CPFIT_MTTKRP_DIRECT_HOST", "1") != "0"


def mttkrp(t: SparseTensor, factors, mode: int, threads: int = 1):
    """Matricized tensor times Khatri-Rao product (kernels.py:46-91).

    out[i, r] = sum over entries with mode index i of value * prod over the
    other modes of factor[i_n, r]; rows with no entries are exactly zero.
    """
    mode = check_mode(mode, t.order)
    factors, rank = _checked_factor_list(factors, t.shape, skip_mode=mode)
    dtype = _compute_dtype(factors)
    on_device = _device_mode(factors)
    torch = _torch()
    dev = [_to_device(f, dtype) for f in factors]
    fin = _FiniteCheck(_named(factors, dev))
    if on_device or not _MTTKRP_DIRECT_HOST:
        out = torch.empty((t.shape[mode], rank), dtype=dtype, device=cuda_device())
    else:
        # numpy operands: the kernel stores its rows straight into the pinned
        # result buffer (each row is written once, 128-byte aligned stores), so
        # the result needs no read-back pass behind whatever else is crossing PCIe
        out = torch.empty((t.shape[mode], rank), dtype=dtype, pin_memory=True)
    if t.nnz == 0:
        out.zero_()
    else:
        vals = t.sorted_values(mode, dtype)
        _lib.check(_lib.load().cpfit_mttkrp(
            t.device_pattern().handle, mode, _dtype_code(dtype), rank, _vp(vals), 1,
            _ptrs(dev), _vp(out), _stream()), "mttkrp")
    if on_device:
        res = out
    elif _MTTKRP_DIRECT_HOST:
        torch.cuda.current_stream().synchronize()
        res = out.numpy()
    else:
        res = to_host_sm(out)
    fin.raise_if_bad()
    return res


def _tttp_slices(rank: int, h_slices, nnz: int, budget_bytes: int):
    """kernels.py:94-102 (validation only: the fused kernel needs no slicing)."""
    if h_slices is None:
        per_slice = max(1, budget_bytes // max(1, nnz * 8))
        h_slices = -(-rank // per_slice)
    h_slices = int(h_slices)
    if not 1 <= h_slices <= rank:
        raise ValueError(f"h_slices must be in [1, rank], got {h_slices}")
    return h_slices


def tttp(t: SparseTensor, factors, h_slices: int | None = None,
         budget_bytes: int = DEFAULT_TTTP_BUDGET_BYTES, threads: int = 1) -> SparseTensor:
    """Tensor-times-tensor product (kernels.py:105-149).

    out value at entry e = t value * sum_r prod over provided modes of
    factors[n][coords[n][e], r]; None slots are skipped.  One fused pass:
    ``h_slices`` is validated but no nnz x R intermediate ever exists.
    """
    factors, rank = _checked_factor_list(factors, t.shape, allow_missing=True)
    if t.nnz == 0:
        check_factor_list(factors, t.shape, allow_missing=True)  # host finiteness scan
        return t
    _tttp_slices(rank, h_slices, t.nnz, budget_bytes)
    dtype = _compute_dtype(factors)
    on_device = _device_mode(factors)
    torch = _torch()
    dev = [_to_device(f, dtype) for f in factors]
    fin = _FiniteCheck(_named(factors, dev))
    vals = t.device_values(dtype)
    out = torch.empty(t.nnz, dtype=dtype, device=cuda_device())
    res = t.with_values(out)
    if on_device:
        _lib.check(_lib.load().cpfit_tttp(
            t.device_pattern().handle, _dtype_code(dtype), rank, _vp(vals), _ptrs(dev),
            _vp(out), _stream()), "tttp")
    else:
        # numpy operands: the reference returns host values -- chunked kernel
        # with the device->host DMA of each chunk overlapping the next chunk,
        # on a library copy stream the caller's stream is NOT joined to: later
        # calls compute while the values drain, and reading `.values` waits
        fin.raise_if_bad()
        host = torch.empty(t.nnz, dtype=dtype, pin_memory=True)
        ev = ctypes.c_void_p()
        _lib.check(_lib.load().cpfit_tttp_host_async(
            t.device_pattern().handle, _dtype_code(dtype), rank, _vp(vals), _ptrs(dev),
            _vp(out), _vp(host), 0, ctypes.byref(ev), _stream()), "tttp_host_async")
        res._pending = _HostValues(res, ev.value, host, out)
        return res
    fin.raise_if_bad()
    return res


class _HostValues:
    """Host values of an asynchronous TTTP: resolves (waits on the copy
    event) on first read; if the tensor is dropped unread, a finalizer waits
    for the DMA before the pinned buffer and device output are released."""

    def __init__(self, owner, event, host, dev):
        import weakref
        self._fin = weakref.finalize(owner, _HostValues._release, event, host, dev)
        self.host = host

    @staticmethod
    def _release(event, host, dev):
        if event:
            _lib.load().cpfit_event_wait(ctypes.c_void_p(event), 1)

    def __call__(self):
        self._fin()  # waits on (and destroys) the event exactly once
        return self.host.numpy()


def sddmm(s: SparseTensor, u, v, threads: int = 1) -> SparseTensor:
    """Sampled dense-dense matrix multiply (kernels.py:152-156)."""
    if s.order != 2:
        raise ValueError(f"sddmm requires an order-2 tensor, got order {s.order}")
    return tttp(s, [u, v], threads=threads)


def _weights_arg(weights: SparseTensor, mode: int, dtype):
    return weights.sorted_values(mode, dtype)


def gram_blocks(weights: SparseTensor, factors, mode: int, row_batches: int = 1,
                stage_rows: int = DEFAULT_STAGE_ROWS, threads: int = 1):
    """Per-row normal-equation matrices (kernels.py:159-212).

    G[i] = sum over entries of row i of weight * h h^T, h = Hadamard product of
    the other modes' factor rows.  ``row_batches`` / ``stage_rows`` are
    validated memory knobs of the reference; the fused kernel needs neither.
    """
    mode = check_mode(mode, weights.order)
    factors, rank = check_factor_list(factors, weights.shape, skip_mode=mode)
    if not 1 <= row_batches:
        raise ValueError("row_batches must be >= 1")
    dtype = _compute_dtype(factors)
    on_device = _device_mode(factors)
    torch = _torch()
    dev = [_to_device(f, dtype) for f in factors]
    gram = torch.empty((weights.shape[mode], rank, rank), dtype=dtype, device=cuda_device())
    if weights.nnz == 0:
        gram.zero_()
    else:
        w = _weights_arg(weights, mode, dtype)
        _lib.check(_lib.load().cpfit_gram(
            weights.device_pattern().handle, mode, _dtype_code(dtype), rank, _vp(w), 1,
            _ptrs(dev), _vp(gram), _stream()), "gram")
    return gram if on_device else to_host(gram)


def gram_matvec(weights: SparseTensor, factors, x, mode: int, row_active=None):
    """Row-wise product with the normal-equation matrices WITHOUT forming them:
    out[i] = G_i x[i] = sum over entries of row i of weight * h (h . x[i]),
    h and G_i as in ``gram_blocks`` (kernels.py:159-212).  One pass over the
    nonzeros (cpfit_gram_matvec); the building block of the implicit-CG ALS
    update (``SolverConfig(als_solver="cg")``).  Not a reference function: its
    oracle is ``einsum('irs,is->ir', gram_blocks(...), x)``.  ``row_active``
    (optional int32 per row, device tensor or array): rows with 0 are skipped
    and return 0."""
    mode = check_mode(mode, weights.order)
    x = check_factor(x, rows=weights.shape[mode], name="x")
    factors, rank = check_factor_list(factors, weights.shape, skip_mode=mode)
    if x.shape[1] != rank:
        raise ValueError(f"x rank {x.shape[1]} does not match factor rank {rank}")
    dtype = _compute_dtype(list(factors) + [x])
    on_device = _device_mode(list(factors) + [x])
    torch = _torch()
    dev = [_to_device(f, dtype) for f in factors]
    dx = _to_device(x, dtype)
    out = torch.empty((weights.shape[mode], rank), dtype=dtype, device=cuda_device())
    act = None
    if row_active is not None:
        act = torch.as_tensor(row_active).to(device=cuda_device(), dtype=torch.int32).contiguous()
        if act.numel() != weights.shape[mode]:
            raise ValueError("row_active must have one entry per row of the mode")
    if weights.nnz == 0:
        out.zero_()
    else:
        w = _weights_arg(weights, mode, dtype)
        _lib.check(_lib.load().cpfit_gram_matvec(
            weights.device_pattern().handle, mode, _dtype_code(dtype), rank, _vp(w), 1,
            _ptrs(dev), _vp(dx), _vp(act), _vp(out), _stream()), "gram_matvec")
    return out if on_device else to_host(out)


def solve_factor(weights: SparseTensor, factors, rhs, mode: int, reg: float = 0.0,
                 row_batches: int = 1, stage_rows: int = DEFAULT_STAGE_ROWS,
                 threads: int = 1, return_gram: bool = False):
    """Per-row regularised normal equations (kernels.py:215-267).

    Solves (G_i + reg I) x_i = rhs_i for every row of ``mode``; empty rows
    solve reg x = rhs (identity when reg == 0, which then requires rhs == 0).

    Raises NumericalError naming the row on a singular system (reg == 0).
    """
    mode = check_mode(mode, weights.order)
    rhs = check_factor(rhs, rows=weights.shape[mode], name="rhs")
    rank = rhs.shape[1]
    factors, frank = check_factor_list(factors, weights.shape, skip_mode=mode)
    if not 1 <= row_batches:
        raise ValueError("row_batches must be >= 1")
    dtype = _compute_dtype(list(factors) + [rhs])
    on_device = _device_mode(list(factors) + [rhs])
    torch = _torch()
    dev = [_to_device(f, dtype) for f in factors]
    drhs = _to_device(rhs, dtype)
    if frank != rank:
        # the reference assembles G first, so negative weights win over this
        if weights.nnz and bool((weights.device_values(dtype) < 0).any()):
            raise ValueError("weights must be nonnegative for normal-equation assembly")
        raise ValueError(f"rhs rank {rank} does not match factor rank {frank}")
    reg = float(reg)
    x = torch.empty((weights.shape[mode], rank), dtype=dtype, device=cuda_device())
    gram = torch.empty((weights.shape[mode], rank, rank), dtype=dtype,
                       device=cuda_device()) if return_gram else None
    w = _weights_arg(weights, mode, dtype) if weights.nnz else None
    bad = ctypes.c_int64(-1)
    pat = weights.device_pattern() if weights.nnz or True else None
    st = _lib.load().cpfit_solve_factor(
        pat.handle, mode, _dtype_code(dtype), rank, _vp(w), 1, _ptrs(dev), _vp(drhs), reg,
        _vp(x), _vp(gram), ctypes.byref(bad), _stream())
    if st == _lib.EEMPTYROW:
        raise NumericalError(f"mode {mode} row {bad.value}: no incident entries and reg=0 "
                             "but right-hand side is nonzero")
    if st == _lib.ESINGULAR:
        raise NumericalError(f"mode {mode} row {bad.value}: singular normal equations "
                             f"(reg={reg})")
    _lib.check(st, "solve_factor")
    if not on_device:
        x = to_host(x)
        gram = to_host(gram) if gram is not None else None
    if return_gram:
        return x, gram
    return x
