"""Cyclops-style façade over the sm_100a kernels (the API north_star names).

The paper writes its completion algorithms against Cyclops' Python interface
(PAPER.md:41-50, 76-83, 108-113, 120-131, 137-139):

    T = ctf.tensor((I, J, K), sp=True)
    S = ctf.TTTP(Omega, [U, V, W])            # or [U, None, W]
    ctf.MTTKRP(T, [rhs, V, W], 0)              # rhs <- einsum('ijk,jr,kr->ir')
    ctf.Solve_Factor(Omega, [U, V, W], rhs, 0, regu)
    a = ctf.einsum('ijk,j,k->i', R, V[:, r], W[:, r])
    b = ctf.einsum('ijk,j,j,k,k->i', Omega, V[:, r], V[:, r], W[:, r], W[:, r])
    T.sample(rate); Omega = getOmega(T)

The reference package (cpfit) has no such interface; its oracle is the
mapping onto cpfit's kernels, which is exactly what this
module does -- every call below runs the same device kernels as
``kernels.tttp`` / ``mttkrp`` / ``solve_factor``, so the results are
bit-identical to those calls.  Only the contractions on the hot path are
recognised by ``einsum``: MTTKRP-shaped ones (one sparse or dense order-N
operand, every other operand a factor matrix ``xr`` or column vector ``x``
on one of its modes, output = the remaining mode) -- repeated vectors on a
mode are multiplied elementwise first (the CCD++ denominator).  Anything else
raises ValueError: general dense contraction planning is Cyclops' own
subsystem, not this path.
"""

from __future__ import annotations

import numpy as np

from .core import RngState, SparseTensor, _is_torch
from .kernels import mttkrp as _mttkrp
from .kernels import solve_factor as _solve_factor
from .kernels import tttp as _tttp


class Tensor:
    """A sparse (``sp=True``) or dense tensor.  Sparse tensors hold a
    SparseTensor (device pattern + values); dense ones hold an array
    (numpy, or a CUDA torch tensor that stays on the device)."""

    __slots__ = ("shape", "sp", "_st", "_dense")

    def __init__(self, shape, sp: bool = False, dtype=np.float64):
        self.shape = tuple(int(d) for d in shape)
        self.sp = bool(sp)
        self._st = SparseTensor(self.shape, np.empty(0, np.uint64), np.empty(0)) if sp else None
        self._dense = None if sp else np.zeros(self.shape, dtype=dtype)

    # -- construction ---------------------------------------------------------
    @classmethod
    def from_sparse(cls, st: SparseTensor) -> "Tensor":
        t = cls.__new__(cls)
        t.shape, t.sp, t._st, t._dense = tuple(st.shape), True, st, None
        return t

    @classmethod
    def from_array(cls, a) -> "Tensor":
        t = cls.__new__(cls)
        t.shape, t.sp, t._st, t._dense = tuple(a.shape), False, None, a
        return t

    def write(self, keys, values) -> None:
        """Set the entries of a sparse tensor: linearized keys (row-major,
        last mode fastest) or a tuple of per-mode coordinate arrays;
        duplicates are summed (the reference's from_coords contract)."""
        if not self.sp:
            raise ValueError("write() with keys is for sparse tensors")
        from .core import delinearize_many, from_coords
        if isinstance(keys, (tuple, list)):
            coords = keys
        else:
            coords = delinearize_many(np.asarray(keys, dtype=np.uint64), self.shape)
        self._st = from_coords(coords, np.asarray(values, dtype=np.float64), self.shape)

    def fill_sp_random(self, lo: float, hi: float, frac: float, seed: int = 0) -> None:
        """Each cell nonzero with probability `frac`, values U(lo, hi)
        (PAPER.md:48); cell space enumerated on the host like gen_low_rank."""
        if not self.sp:
            raise ValueError("fill_sp_random is for sparse tensors")
        g = RngState(seed).generator()
        total = int(np.prod(self.shape, dtype=np.float64))
        keys = np.flatnonzero(g.random(total) < frac).astype(np.uint64)
        vals = lo + (hi - lo) * g.random(keys.size)
        self._st = SparseTensor(self.shape, keys, vals, validate=False)

    # -- access ---------------------------------------------------------------
    @property
    def sparse(self) -> SparseTensor:
        if not self.sp:
            raise ValueError("not a sparse tensor")
        return self._st

    @property
    def array(self):
        return self._st.values if self.sp else self._dense

    def read_all(self):
        """(keys, values) of a sparse tensor; the array of a dense one."""
        if self.sp:
            return self._st.keys, self._st.values
        return self._dense

    def copy(self) -> "Tensor":
        if self.sp:
            return Tensor.from_sparse(self._st.with_values(self._st.values.copy()))
        d = self._dense
        return Tensor.from_array(d.clone() if _is_torch(d) else np.array(d, copy=True))

    def sample(self, rate: float, rng: RngState | None = None) -> None:
        """Keep each entry with probability `rate`, in place (
        device Philox, bit-exact with SparseTensor.sample)."""
        if not self.sp:
            raise ValueError("sample is for sparse tensors")
        self._st = self._st.sample(rate, rng if rng is not None else RngState(0))

    def norm2(self) -> float:
        v = self.array
        if _is_torch(v):
            return float(v.double().norm())
        return float(np.linalg.norm(np.asarray(v).ravel()))

    def __sub__(self, other):
        if self.sp and isinstance(other, Tensor) and other.sp:
            a, b = self._st, other._st
            if a.nnz != b.nnz or not np.array_equal(a.keys, b.keys):
                raise ValueError("sparse difference needs a shared sparsity pattern")
            return Tensor.from_sparse(a.with_values(a.values - b.values))
        raise ValueError("only pattern-sharing sparse differences are on this path")

    def __repr__(self) -> str:
        kind = f"sparse nnz={self._st.nnz}" if self.sp else "dense"
        return f"ctf.Tensor({self.shape}, {kind})"


def tensor(shape, sp: bool = False, dtype=np.float64) -> Tensor:
    """ctf.tensor(shape, sp=...)."""
    return Tensor(shape, sp=sp, dtype=dtype)


def getOmega(T: Tensor) -> Tensor:
    """Unit-valued tensor on T's pattern (observation_mask)."""
    return Tensor.from_sparse(T.sparse.observation_mask())


def _mat(x):
    """Factor operand -> 2-D array (a vector is one column)."""
    if x is None:
        return None
    a = x.array if isinstance(x, Tensor) else x
    if a.ndim == 1:
        return a.reshape(-1, 1)
    return a


def _assign(dst, value) -> None:
    """Write a result into the caller's operand (Cyclops writes in place)."""
    if isinstance(dst, Tensor):
        tgt = dst.array
    else:
        tgt = dst
    if _is_torch(tgt):
        import torch
        v = value if _is_torch(value) else torch.from_numpy(np.asarray(value))
        tgt.copy_(v.reshape(tgt.shape).to(tgt.dtype))
    elif isinstance(dst, Tensor) and not dst.sp:
        if _is_torch(value):
            value = value.cpu().numpy()
        dst._dense = np.asarray(value).reshape(dst.shape).copy()
    else:
        if _is_torch(value):
            value = value.cpu().numpy()
        np.copyto(tgt, np.asarray(value).reshape(tgt.shape))


def TTTP(Omega: Tensor, factors) -> Tensor:
    """S = ctf.TTTP(Omega, [U, V, W, Z]) with None slots skipped
     -> kernels.tttp."""
    return Tensor.from_sparse(_tttp(Omega.sparse, [_mat(f) for f in factors]))


def MTTKRP(T: Tensor, mats, mode: int) -> None:
    """ctf.MTTKRP(T, [rhs, V, W], 0): mats[mode] <- MTTKRP of T with the other
    operands -> kernels.mttkrp.  Vectors act as R=1."""
    fs = [None if n == mode else _mat(m) for n, m in enumerate(mats)]
    _assign(mats[mode], _mttkrp(T.sparse, fs, mode))


def Solve_Factor(Omega: Tensor, mats, rhs, mode: int, regu: float) -> None:
    """ctf.Solve_Factor(Omega, [U, V, W], rhs, 0, regu): mats[mode] <- the
    regularised per-row normal-equation solutions ->
    kernels.solve_factor."""
    fs = [None if n == mode else _mat(m) for n, m in enumerate(mats)]
    _assign(mats[mode], _solve_factor(Omega.sparse, fs, _mat(rhs), mode, reg=float(regu)))


# ---- einsum ------------------------------------------------------------------

def plan_einsum(spec: str, ndims):
    """Parse an MTTKRP-shaped contraction.  Returns (mode, rank_letter, groups)
    where groups[n] lists the operand positions (1..) applied to mode n of
    operand 0 (empty for the output mode).  Raises ValueError otherwise.
    Pure host logic (tested without a GPU)."""
    spec = spec.replace(" ", "")
    if "->" not in spec:
        raise ValueError("einsum needs an explicit output ('->')")
    lhs, out = spec.split("->")
    terms = lhs.split(",")
    if len(terms) != len(ndims):
        raise ValueError("operand count does not match the subscripts")
    t0 = terms[0]
    if len(set(t0)) != len(t0):
        raise ValueError("repeated index on the tensor operand")
    for term, nd in zip(terms, ndims):
        if len(term) != nd:
            raise ValueError(f"subscripts {term!r} do not match an operand of order {nd}")
    rank_letters = {c for term in terms[1:] for c in term if c not in t0}
    if len(rank_letters) > 1:
        raise ValueError("at most one rank index is supported")
    r = next(iter(rank_letters)) if rank_letters else None
    if r is not None and r in t0:
        raise ValueError("the rank index must not index the tensor")
    out_modes = [c for c in out if c in t0]
    if len(out_modes) != 1 or (r is not None and out != out_modes[0] + r and out != r + out_modes[0]) \
            or (r is None and out != out_modes[0]):
        raise ValueError(f"output {out!r} is not one tensor mode (plus the rank index): "
                         "only MTTKRP-shaped contractions are on this path")
    if r is not None and out != out_modes[0] + r:
        raise ValueError("output must be laid out (mode, rank)")
    mode = t0.index(out_modes[0])
    groups = [[] for _ in t0]
    for k, term in enumerate(terms[1:], start=1):
        idx = [c for c in term if c in t0]
        rest = [c for c in term if c not in t0]
        if len(idx) != 1 or (rest and rest != [r]) or (r is not None and not rest):
            raise ValueError(f"operand {term!r} must be a factor on one tensor mode"
                             + (f" with the rank index {r!r}" if r else ""))
        if r is not None and term != idx[0] + r:
            raise ValueError(f"factor {term!r} must be laid out (mode, rank)")
        groups[t0.index(idx[0])].append(k)
    for n, g in enumerate(groups):
        if n == mode and g:
            raise ValueError("the output mode cannot also be contracted")
        if n != mode and not g:
            raise ValueError(f"mode {t0[n]!r} is not contracted by any factor")
    return mode, r, groups


def einsum(spec: str, *operands):
    """MTTKRP-shaped einsum: 'ijk,jr,kr->ir', 'ijk,j,k->i',
    'ijk,j,j,k,k->i', ... on a sparse Tensor / SparseTensor (kernels.mttkrp)
    or an order-3 dense CUDA tensor (dense MTTKRP kernels)."""
    X = operands[0]
    st = X.sparse if isinstance(X, Tensor) and X.sp else (X if isinstance(X, SparseTensor)
                                                           else None)
    xd = None if st is not None else (X.array if isinstance(X, Tensor) else X)
    order = len(st.shape) if st is not None else xd.ndim
    ndims = [order] + [(o.array if isinstance(o, Tensor) else o).ndim for o in operands[1:]]
    mode, r, groups = plan_einsum(spec, ndims)
    mats = []
    for n, g in enumerate(groups):
        if n == mode:
            mats.append(None)
            continue
        f = _mat(operands[g[0]])
        for k in g[1:]:
            f = f * _mat(operands[k])   # repeated vectors on a mode: elementwise first
        mats.append(f)
    if st is not None:
        res = _mttkrp(st, mats, mode)
    else:
        from .dense import dense_mttkrp
        if not _is_torch(xd) or order != 3:
            raise ValueError("dense einsum runs on order-3 CUDA tensors")
        import torch
        mats = [None if m is None else (m if _is_torch(m) else torch.from_numpy(m)).to(
            device=xd.device, dtype=xd.dtype) for m in mats]
        res = dense_mttkrp(xd, mats, mode)
    return res if r is not None else res.reshape(-1)


__all__ = ["Tensor", "tensor", "getOmega", "TTTP", "MTTKRP", "Solve_Factor", "einsum",
           "plan_einsum"]
