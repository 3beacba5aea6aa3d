"""Multi-GPU sharding of the completion sweeps (one process per GPU, NCCL).

SURVEY.md 8(e): ALS shards *rows*.  For every mode n the rows of mode n are
cut into P contiguous blocks balanced by the nonzero prefix sum (Zipf rows
make equal row counts useless); rank p keeps a *mode shard*: the nonzeros
whose mode-n index lies in its block, with that coordinate rebased to the
block (shape[n] = block rows) and every other coordinate global.  Right-hand
side (MTTKRP), Gram and solve are all row-local, so one mode update is:
local MTTKRP + fused Gram/solve on the shard, then one uneven all-gather of
the updated I_n x R rows: one broadcast per block from its owner into the
replicated factor (NCCL over NVLink/NVSwitch moves exactly I_n x R values,
never a block padded to the largest one).  Blocks balance a cost model, not
just nonzeros: a row costs its nonzeros (Gram + right-hand side) plus a
per-row term for the R x R solve and the Gram store/load
(``als_row_weight``).  No other exchange: factors are replicated.

SGD shards *nonzeros* (contiguous key ranges); the device Philox sampler uses
the global entry index as its counter, so the union of the shard samples is
the single-device sample bit for bit, and the per-mode gradients are summed
with one all-reduce (``ShardedSGD``).  CCD++ shards nonzeros too and
all-reduces the per-row (num, den) sums of every (r, mode) column update
(``ShardedCCD``).

The partition / shard / assembly logic is backend-neutral: ``LocalBackend``
objects supply the row-local compute.  ``DeviceBackend`` runs the CUDA
kernels; tests (tests/test_dist.py, gloo, world size 2 on CPU) plug in the CPU
oracle to check the distributed algebra without a GPU.
"""

from __future__ import annotations

import math

import numpy as np


def als_row_weight(rank: int) -> float:
    """Cost of one row's solve + Gram store/load in units of one nonzero's
    Gram + right-hand-side work.  Measured at cfg 3 (R = 32, one B200):
    fused Gram + rhs 6.9 ms / 1.005e8 nnz = 0.069 ns per nonzero; batched
    Cholesky 2.45 ms + 2 x 3.9 GB of G traffic ~ 3.65 ms / 480,189 rows =
    7.6 ns per row -> ~110 at R = 32.  The solve grows like R^3 and the
    per-nonzero Gram like R^2, so the ratio scales ~linearly in R."""
    return 3.4 * float(rank)


def row_partition(row_counts, parts: int, row_weight: float = 0.0):
    """Contiguous row blocks [lo, hi) balanced by the prefix sum of the row
    cost nnz_i + row_weight (row_weight 0: by nonzeros only)."""
    counts = np.asarray(row_counts, dtype=np.float64)
    prefix = np.concatenate([[0.0], np.cumsum(counts + float(row_weight))])
    total = float(prefix[-1])
    bounds = [0]
    for p in range(1, parts):
        target = total * p / parts
        r = int(np.searchsorted(prefix, target, side="left"))
        r = max(bounds[-1], min(r, counts.size))
        bounds.append(r)
    bounds.append(counts.size)
    return [(bounds[i], bounds[i + 1]) for i in range(parts)]


def nnz_partition(nnz: int, parts: int, align: int = 4):
    """Contiguous nonzero ranges (aligned so Philox blocks of 4 draws are not
    split across ranks; any split would still be bit-exact)."""
    out = []
    for p in range(parts):
        lo = (nnz * p // parts) // align * align
        hi = nnz if p == parts - 1 else (nnz * (p + 1) // parts) // align * align
        out.append((lo, hi))
    return out


def shard_keys(coords, shape, mode: int, lo: int, hi: int, xp=np):
    """Select entries with lo <= i_mode < hi and re-linearize with the mode
    rebased; returns (shard shape, keys, selection mask).  ``xp`` is numpy or
    torch (coords as int64 arrays of the backend)."""
    sel = (coords[mode] >= lo) & (coords[mode] < hi)
    sshape = list(shape)
    sshape[mode] = max(hi - lo, 1)
    key = None
    for n, d in enumerate(sshape):
        c = coords[n][sel]
        if n == mode:
            c = c - lo
        key = c if key is None else key * d + c
    return tuple(sshape), key, sel


def pad_rows(x, rows: int, xp=np):  # kept for callers that pad explicitly
    if x.shape[0] == rows:
        return x
    if xp is np:
        out = np.zeros((rows,) + tuple(x.shape[1:]), dtype=x.dtype)
    else:
        out = xp.zeros((rows,) + tuple(x.shape[1:]), dtype=x.dtype, device=x.device)
    out[: x.shape[0]] = x
    return out


class ShardedALS:
    """Row-sharded ALS sweeps over a process group.

    backend: object with
      make_shard(shape, keys, values) -> handle
      als_mode(handle, factors, mode, reg) -> updated rows of the block
      to_comm(x) / from_comm(x) -> tensors for torch.distributed
      xp -> numpy or torch (for shard_keys / padding)
    """

    def __init__(self, coords, values, shape, reg, backend, group=None, rank_r: int = 32,
                 row_weight: float | None = None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.shape = tuple(shape)
        self.reg = float(reg)
        self.backend = backend
        self.row_weight = als_row_weight(rank_r) if row_weight is None else float(row_weight)
        xp = backend.xp
        self.blocks = []
        self.shards = []
        for mode, d in enumerate(self.shape):
            if xp is np:
                counts = np.bincount(coords[mode], minlength=d)
            else:
                counts = xp.bincount(coords[mode], minlength=d).cpu().numpy()
            blocks = row_partition(counts, self.world, self.row_weight)
            lo, hi = blocks[self.rank]
            sshape, keys, sel = shard_keys(coords, self.shape, mode, lo, hi, xp)
            self.blocks.append(blocks)
            self.shards.append(backend.make_shard(sshape, keys, values[sel]))

    def mode_update(self, factors, mode: int):
        """Local update of this rank's rows, then an uneven all-gather: the
        owner of each block broadcasts exactly its rows into the replicated
        factor (I_n x R values on the wire, no padding)."""
        blocks = self.blocks[mode]
        lo, hi = blocks[self.rank]
        rows = self.backend.to_comm(
            self.backend.als_mode(self.shards[mode], factors, mode, self.reg, lo, hi))
        full = self.backend.empty_comm((self.shape[mode],) + tuple(rows.shape[1:]), rows)
        for p, (a, b) in enumerate(blocks):
            if b == a:
                continue
            view = full[a:b]
            if p == self.rank:
                view.copy_(rows)
            if self.world > 1:
                src = p if self.group is None else self.dist.get_global_rank(self.group, p)
                self.dist.broadcast(view, src=src, group=self.group)
        factors[mode] = self.backend.from_comm(full)

    def exchanged_bytes(self, mode: int, rank_r: int, itemsize: int = 8) -> int:
        """Bytes one mode's gather puts on the wire (sum of the blocks)."""
        return sum(b - a for a, b in self.blocks[mode]) * rank_r * itemsize

    def sweep(self, factors):
        for mode in range(len(self.shape)):
            self.mode_update(factors, mode)
        return factors


class ShardedCCD:
    """Nonzero-sharded CCD++ sweeps: each rank keeps a
    contiguous key range of the entries and its slice of the residual; per
    (r, mode) the per-row (num, den) sums of the shard are all-reduced (2 I_n
    values) and every rank computes the identical new column; the shard's
    rhat (residual with column r added back) is re-formed once per column.
    optim.py:235-268 least-squares branch.

    backend: ccd_begin(shard, factors) -> state; ccd_numden(shard, state, r,
    mode) -> comm tensor (2 I_n); ccd_apply(shard, state, r, mode, numden, reg);
    ccd_end(state, factors); make_nnz_shard(shape, keys, values)."""

    def __init__(self, keys, values, shape, reg, backend, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.shape = tuple(shape)
        self.reg = float(reg)
        self.backend = backend
        self.lo, self.hi = nnz_partition(len(keys), self.world)[self.rank]
        self.shard = backend.make_nnz_shard(self.shape, keys[self.lo:self.hi],
                                            values[self.lo:self.hi])

    def sweep(self, factors):
        b = self.backend
        state = b.ccd_begin(self.shard, factors)
        rank = factors[0].shape[1]
        for r in range(rank):
            for mode in range(len(self.shape)):
                nd = b.ccd_numden(self.shard, state, r, mode)
                if self.world > 1:
                    self.dist.all_reduce(nd, group=self.group)
                b.ccd_apply(self.shard, state, r, mode, nd, self.reg)
        b.ccd_end(state, factors)
        return factors


class ShardedSGD:
    """Nonzero-sharded SGD steps: rank p samples its key range
    with the global Philox counter (the union of the shard samples is the
    single-device sample bit for bit), computes the least-squares gradient
    MTTKRPs of its sample, the gradients are summed with one all-reduce per
    mode and every rank applies the identical update (optim.py:300-330).

    backend: make_nnz_shard; sgd_grads(shard, factors, rate, rng, counter_offset)
    -> list of comm tensors; sgd_apply(factors, grads, step, shrink)."""

    def __init__(self, keys, values, shape, backend, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.shape = tuple(shape)
        self.backend = backend
        self.lo, self.hi = nnz_partition(len(keys), self.world)[self.rank]
        self.shard = backend.make_nnz_shard(self.shape, keys[self.lo:self.hi],
                                            values[self.lo:self.hi])

    def step(self, factors, rate: float, step: float, reg: float, rng):
        b = self.backend
        grads = b.sgd_grads(self.shard, factors, rate, rng, self.lo)
        if self.world > 1:
            for g in grads:
                self.dist.all_reduce(g, group=self.group)
        b.sgd_apply(factors, grads, step, 2.0 * step * reg * rate)
        return factors


class DeviceBackend:
    """CUDA kernels + NCCL (factors are CUDA tensors)."""

    def __init__(self, als_solver: str = "direct", cg_tol: float = 5e-3, cg_max: int = 30):
        import torch
        self.torch = torch
        self.xp = torch
        if als_solver not in ("direct", "cg"):
            raise ValueError(f"unknown als_solver {als_solver!r}")
        self.als_solver = als_solver
        self.cg_tol = float(cg_tol)
        self.cg_max = int(cg_max)

    def make_shard(self, shape, keys, values):
        from .core import SparseTensor
        return SparseTensor.from_device(shape, keys.contiguous(), values.contiguous())

    def als_mode(self, shard, factors, mode, reg, lo, hi):
        """Rows lo..hi of the updated factor: MTTKRP + Gram + solve on the shard,
        with the shard's own (rebased) mode factor slot unused -- or, with
        als_solver="cg", the Gram-free per-row CG update warm-started from the
        block's current rows (SolverConfig.als_solver)."""
        from .optim import _als_mode_cg_device, _als_mode_device
        if self.als_solver == "cg":
            local = list(factors)
            local[mode] = factors[mode][lo:hi].contiguous()
            x, _, _ = _als_mode_cg_device(shard, local, mode, reg, self.cg_tol, self.cg_max)
            return x
        return _als_mode_device(shard, factors, mode, reg, row_offset=lo)

    def make_nnz_shard(self, shape, keys, values):
        from .core import SparseTensor
        return SparseTensor.from_device(shape, keys.contiguous(), values.contiguous())

    # -- CCD++ (cpfit_ccd_step with numden / cpfit_ccd_finalize / cpfit_ccd_fold) --
    def ccd_begin(self, shard, factors):
        torch = self.torch
        from .losses import tttp_affine
        from .optim import _ccd_col_ptrs, _ccd_lean, _ccd_rhat_copies
        cols = [f.t().contiguous() for f in factors]  # R x I_n
        resid = tttp_affine(shard, factors, -1.0, 1.0, torch.float64)  # t - model
        lean = _ccd_lean(shard)
        old = [torch.empty(d, dtype=torch.float64, device=resid.device) for d in shard.shape]
        return {"cols": cols, "rh": _ccd_rhat_copies(shard, resid, lean), "lean": lean,
                "old": old, "old_ptrs": _ccd_col_ptrs(old), "prev": None, "shard": shard}

    def ccd_numden(self, shard, state, r, mode):
        """Local (num, den) of column r on `mode`; the pass first re-forms the
        shard's rhat copy of this mode for column r (csrc/ccd.cu)."""
        import ctypes

        from . import _lib
        from .optim import _ccd_col_ptrs, _stream
        keep, ptrs = _ccd_col_ptrs(state["cols"], r)
        if mode == 0:
            state["cur"] = (keep, ptrs)
            for n, o in enumerate(state["old"]):
                o.copy_(state["cols"][n][r])
        nd = self.torch.empty(2 * shard.shape[mode], dtype=self.torch.float64,
                              device=state["rh"][0].device)
        sub = state["prev"][1] if state["prev"] is not None else None
        if state["lean"]:
            f = mode == 0
            args = (state["rh"][0], 0, sub if f else None, ptrs if f else None)
        else:
            args = (state["rh"][mode], 1, sub, state["old_ptrs"][1])
        _lib.check(_lib.load().cpfit_ccd_step(
            shard.device_pattern().handle, mode, ptrs, ctypes.c_void_p(args[0].data_ptr()),
            args[1], args[2], args[3], 0.0, ctypes.c_void_p(nd.data_ptr()), _stream()),
            "ccd_step")
        return nd

    def ccd_apply(self, shard, state, r, mode, nd, reg):
        import ctypes

        from . import _lib
        from .optim import _stream
        col = state["cols"][mode][r]
        _lib.check(_lib.load().cpfit_ccd_finalize(
            col.numel(), ctypes.c_void_p(nd.data_ptr()), float(reg),
            ctypes.c_void_p(col.data_ptr()), _stream()), "ccd_finalize")
        if mode == shard.order - 1:
            state["prev"] = state["cur"]

    def ccd_end(self, state, factors):
        import ctypes

        from . import _lib
        from .optim import _stream
        if state["prev"] is not None and state["rh"][0].numel():
            _lib.check(_lib.load().cpfit_ccd_fold(
                state["shard"].device_pattern().handle, -1, state["prev"][1], None,
                ctypes.c_void_p(state["rh"][0].data_ptr()), _stream()), "ccd_fold")
        for n, c in enumerate(state["cols"]):
            factors[n] = c.t().contiguous()

    # -- SGD --
    def sgd_grads(self, shard, factors, rate, rng, counter_offset):
        from .optim import _sgd_grads_device
        grads, _ = _sgd_grads_device(shard, factors, rate, rng, factors[0].dtype,
                                     counter_offset=counter_offset)
        return grads

    def sgd_apply(self, factors, grads, step, shrink):
        from .optim import _sgd_apply_device
        _sgd_apply_device(factors, grads, step, shrink)

    def to_comm(self, x):
        return x.contiguous()

    def from_comm(self, x):
        return x.contiguous()

    def empty_comm(self, shape, like):
        return self.torch.empty(shape, dtype=like.dtype, device=like.device)

    def cat(self, parts):
        return self.torch.cat(parts, 0)


def als_strong_scaling_rows(blocks):
    """Largest block share (the load imbalance bound of a sharded sweep)."""
    sizes = [b - a for a, b in blocks]
    return max(sizes) / max(1, sum(sizes)) * len(sizes)


__all__ = ["row_partition", "als_row_weight", "nnz_partition", "shard_keys", "ShardedALS",
           "ShardedCCD", "ShardedSGD", "DeviceBackend", "pad_rows", "als_strong_scaling_rows",
           "math"]
