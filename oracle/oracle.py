"""CPU oracle for the TTTP / MTTKRP / Gram-solve / ALS / CCD++ / SGD path.

TEST INFRASTRUCTURE ONLY -- imported by ``tests/``, ``__graft_entry__.smoke()``
and ``bench.py`` (its ``cpu_baseline`` leg and ``--impl reference``), always as
the checker or the CPU yardstick, never as the thing measured or shipped.  The
product package ``paper_1910_02371_b200`` never imports it.

The numeric kernels live in ``cpfit_oracle.c`` (restating the reference's
numba loops, ``/root/reference/pkg/src/cpfit/_jit.py:35-59``); this module
restates the reference's driver logic on top of them, citing file:line of the
reference package ``cpfit`` (abbreviated ``core.py`` = ``pkg/src/cpfit/core.py``
and so on).  The oracle is pinned against vectors produced by the reference
itself (``tests/golden/make_golden.py``; checked in ``tests/test_oracle.py``).
"""

from __future__ import annotations

import ctypes
import math
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None

_i64p = ctypes.POINTER(ctypes.c_int64)
_u64p = ctypes.POINTER(ctypes.c_uint64)
_f64p = ctypes.POINTER(ctypes.c_double)


def build() -> str:
    """Compile liboracle.so with the committed Makefile (gcc + OpenMP)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        src = os.path.join(_HERE, "cpfit_oracle.c")
        if (not os.path.exists(_LIB_PATH)
                or os.path.getmtime(_LIB_PATH) < os.path.getmtime(src)):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        L.oracle_set_threads.argtypes = [ctypes.c_int]
        L.oracle_set_threads.restype = ctypes.c_int
        L.oracle_delinearize.argtypes = [ctypes.c_int, _i64p, ctypes.c_int64, _u64p, _i64p]
        L.oracle_linearize.argtypes = [ctypes.c_int, _i64p, ctypes.c_int64, _i64p, _u64p]
        L.oracle_counting_sort.argtypes = [ctypes.c_int64, _i64p, ctypes.c_int64, _i64p, _i64p]
        L.oracle_tttp.argtypes = [ctypes.c_int, ctypes.c_int64, ctypes.c_int, _i64p, _f64p,
                                  ctypes.POINTER(ctypes.c_void_p), _f64p]
        L.oracle_mttkrp.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int64, ctypes.c_int,
                                    ctypes.c_int64, _i64p, _f64p, _i64p, _i64p,
                                    ctypes.POINTER(ctypes.c_void_p), _f64p]
        L.oracle_gram.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int64, ctypes.c_int,
                                  ctypes.c_int64, _i64p, _f64p, _i64p, _i64p,
                                  ctypes.POINTER(ctypes.c_void_p), _f64p]
        L.oracle_gram.restype = ctypes.c_int
        L.oracle_solve.argtypes = [ctypes.c_int64, ctypes.c_int, _f64p, _f64p, _i64p,
                                   ctypes.c_double, _f64p, _i64p]
        L.oracle_solve.restype = ctypes.c_int
        L.oracle_philox_uniform.argtypes = [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_int64,
                                            ctypes.c_int64, _f64p]
        L.oracle_sample.argtypes = [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_int64,
                                    ctypes.c_double, _i64p]
        L.oracle_sample.restype = ctypes.c_int64
        L.oracle_ccd_sweep.argtypes = [ctypes.c_int, _i64p, ctypes.c_int64, ctypes.c_int,
                                       _i64p, _f64p, ctypes.POINTER(ctypes.c_void_p),
                                       ctypes.c_double]
        _lib = L
    return _lib


def set_threads(n: int) -> int:
    return int(lib().oracle_set_threads(int(n)))


def _p(a, t):
    return a.ctypes.data_as(t)


def _ptr_array(arrays):
    arr = (ctypes.c_void_p * len(arrays))()
    for i, a in enumerate(arrays):
        arr[i] = None if a is None else a.ctypes.data
    return arr


class OracleError(Exception):
    """Raised with (kind, row) where the reference raises NumericalError/ValueError."""

    def __init__(self, kind: str, row: int = -1, msg: str = ""):
        super().__init__(msg or f"{kind} row {row}")
        self.kind = kind
        self.row = row


# ---------------------------------------------------------------------------
# layout (core.py)

def delinearize(keys, dims) -> np.ndarray:
    """core.py:93-102 -> (order, m) int64 coordinates."""
    keys = np.ascontiguousarray(keys, dtype=np.uint64)
    dims_a = np.ascontiguousarray(dims, dtype=np.int64)
    out = np.empty((len(dims), keys.size), dtype=np.int64)
    lib().oracle_delinearize(len(dims), _p(dims_a, _i64p), keys.size, _p(keys, _u64p),
                             _p(out, _i64p))
    return out


def linearize(coords, dims) -> np.ndarray:
    """core.py:78-90."""
    coords = np.ascontiguousarray(coords, dtype=np.int64)
    dims_a = np.ascontiguousarray(dims, dtype=np.int64)
    keys = np.empty(coords.shape[1], dtype=np.uint64)
    lib().oracle_linearize(len(dims), _p(dims_a, _i64p), keys.size, _p(coords, _i64p),
                           _p(keys, _u64p))
    return keys


def counting_sort(idx, dim):
    """core.py:234-249 -> (perm int64[m], offsets int64[dim+1])."""
    idx = np.ascontiguousarray(idx, dtype=np.int64)
    perm = np.empty(idx.size, dtype=np.int64)
    offsets = np.empty(int(dim) + 1, dtype=np.int64)
    lib().oracle_counting_sort(idx.size, _p(idx, _i64p), int(dim), _p(perm, _i64p),
                               _p(offsets, _i64p))
    return perm, offsets


@dataclass
class OTensor:
    """Oracle-side sparse tensor: sorted uint64 keys + f64 values (core.py:105-131)."""

    shape: tuple
    keys: np.ndarray
    values: np.ndarray
    _coords: np.ndarray | None = None
    _groups: dict = field(default_factory=dict)

    @property
    def order(self):
        return len(self.shape)

    @property
    def nnz(self):
        return int(self.keys.size)

    def coords(self):
        if self._coords is None:
            self._coords = delinearize(self.keys, self.shape)
        return self._coords

    def mode_group(self, mode):
        hit = self._groups.get(mode)
        if hit is None:
            hit = counting_sort(self.coords()[mode], self.shape[mode])
            self._groups[mode] = hit
        return hit

    def with_values(self, values):
        out = OTensor(self.shape, self.keys, np.ascontiguousarray(values, dtype=np.float64))
        out._coords = self._coords
        out._groups = self._groups
        return out


def from_coords(coord_arrays, values, shape) -> OTensor:
    """core.py:208-231: stable sort by key, duplicates summed in stable order."""
    keys = linearize(np.stack([np.asarray(c, dtype=np.int64) for c in coord_arrays]), shape)
    values = np.ascontiguousarray(values, dtype=np.float64)
    order = np.argsort(keys, kind="stable")
    keys, values = keys[order], values[order]
    if keys.size:
        starts = np.flatnonzero(np.concatenate(([True], keys[1:] != keys[:-1])))
        if starts.size != keys.size:
            values = np.add.reduceat(values, starts)
            keys = keys[starts]
    return OTensor(tuple(int(d) for d in shape), keys, values)


# ---------------------------------------------------------------------------
# kernels (kernels.py)

def _factors64(factors):
    return [None if f is None else np.ascontiguousarray(f, dtype=np.float64)
            for f in factors]


def tttp(t: OTensor, factors) -> np.ndarray:
    """kernels.py:105-149 / _jit.py:49-59 -> output values (same keys)."""
    fs = _factors64(factors)
    rank = next(f.shape[1] for f in fs if f is not None)
    out = np.empty(t.nnz)
    if t.nnz == 0:
        return out
    coords = t.coords()
    lib().oracle_tttp(t.order, t.nnz, rank, _p(coords, _i64p), _p(t.values, _f64p),
                      _ptr_array(fs), _p(out, _f64p))
    return out


def mttkrp(t: OTensor, factors, mode: int) -> np.ndarray:
    """kernels.py:46-91 / _jit.py:35-47."""
    fs = _factors64(factors)
    fs[mode] = None
    rank = next(f.shape[1] for f in fs if f is not None)
    out = np.zeros((t.shape[mode], rank))
    if t.nnz == 0:
        return out
    perm, offsets = t.mode_group(mode)
    lib().oracle_mttkrp(t.order, mode, t.nnz, rank, t.shape[mode], _p(t.coords(), _i64p),
                        _p(t.values, _f64p), _p(perm, _i64p), _p(offsets, _i64p),
                        _ptr_array(fs), _p(out, _f64p))
    return out


def gram_blocks(w: OTensor, factors, mode: int) -> np.ndarray:
    """kernels.py:159-212 (unit weights = observation mask for LS ALS)."""
    fs = _factors64(factors)
    fs[mode] = None
    rank = next(f.shape[1] for f in fs if f is not None)
    gram = np.zeros((w.shape[mode], rank, rank))
    if w.nnz == 0:
        if np.any(w.values < 0):
            raise OracleError("negative_weights")
        return gram
    perm, offsets = w.mode_group(mode)
    st = lib().oracle_gram(w.order, mode, w.nnz, rank, w.shape[mode], _p(w.coords(), _i64p),
                           _p(w.values, _f64p), _p(perm, _i64p), _p(offsets, _i64p),
                           _ptr_array(fs), _p(gram, _f64p))
    if st:
        raise OracleError("negative_weights")
    return gram


def solve_factor(w: OTensor, factors, rhs, mode: int, reg: float = 0.0,
                 return_gram: bool = False):
    """kernels.py:215-267 (LU restatement of LAPACK gesv, kernels.py:259)."""
    rhs = np.ascontiguousarray(rhs, dtype=np.float64)
    gram = gram_blocks(w, factors, mode)
    if w.nnz:
        _, offsets = w.mode_group(mode)
    else:
        offsets = np.zeros(w.shape[mode] + 1, dtype=np.int64)
    x = np.empty_like(rhs)
    bad = ctypes.c_int64(-1)
    st = lib().oracle_solve(w.shape[mode], rhs.shape[1], _p(gram, _f64p), _p(rhs, _f64p),
                            _p(offsets, _i64p), float(reg), _p(x, _f64p), ctypes.byref(bad))
    if st == 2:
        raise OracleError("empty_row", bad.value)
    if st == 3:
        raise OracleError("singular", bad.value)
    return (x, gram) if return_gram else x


def model_values(factors, coords) -> np.ndarray:
    """core.py:252-266 (numpy restatement, column blocks of 32)."""
    n_entries = coords.shape[1]
    rank = factors[0].shape[1]
    out = np.zeros(n_entries)
    for lo in range(0, rank, 32):
        hi = min(lo + 32, rank)
        prod = factors[0][coords[0], lo:hi].copy()
        for n in range(1, len(factors)):
            prod *= factors[n][coords[n], lo:hi]
        out += prod.sum(axis=1)
    return out


# ---------------------------------------------------------------------------
# sampling (core.py:25-46, 173-183)

def philox_key(seed: int, path: tuple = ()) -> tuple[int, int]:
    """Philox key of RngState(seed, path).generator() (core.py:38-40)."""
    ss = np.random.SeedSequence(entropy=seed, spawn_key=tuple(path))
    key = np.random.Philox(ss).state["state"]["key"]
    return int(key[0]), int(key[1])


def uniform(seed: int, path: tuple, n: int, start: int = 0) -> np.ndarray:
    k0, k1 = philox_key(seed, path)
    out = np.empty(n)
    lib().oracle_philox_uniform(k0, k1, start, n, _p(out, _f64p))
    return out


def sample_positions(t: OTensor, rate: float, seed: int, path: tuple) -> np.ndarray:
    if not 0.0 < rate <= 1.0:
        raise OracleError("rate")
    k0, k1 = philox_key(seed, path)
    kept = np.empty(max(t.nnz, 1), dtype=np.int64)
    c = lib().oracle_sample(k0, k1, t.nnz, float(rate), _p(kept, _i64p))
    return kept[:c].copy()


def sample(t: OTensor, rate: float, seed: int, path: tuple) -> OTensor:
    kept = sample_positions(t, rate, seed, path)
    return OTensor(t.shape, t.keys[kept], t.values[kept])


# ---------------------------------------------------------------------------
# drivers (optim.py)

def init_factors(shape, rank: int, seed: int, path=(0,)):
    """optim.py:113-146 init_state, default uniform law on [0, 1/sqrt(R)]."""
    ss = np.random.SeedSequence(entropy=seed, spawn_key=tuple(path))
    g = np.random.Generator(np.random.Philox(ss))
    scale = 1.0 / math.sqrt(rank)
    return [g.random((d, rank)) * scale for d in shape]


def als_sweep(t: OTensor, factors, reg: float):
    """optim.py:180-207 least-squares branch; returns per-mode (gram, rhs)."""
    mask = t.with_values(np.ones(t.nnz))
    grams, rhss = [], []
    for mode in range(t.order):
        rhs = mttkrp(t, factors, mode)
        new, gram = solve_factor(mask, factors, rhs, mode, reg=reg, return_gram=True)
        factors[mode] = new
        grams.append(gram)
        rhss.append(rhs)
    return grams, rhss


def ccd_sweep(t: OTensor, factors, reg: float):
    """optim.py:235-268 least-squares branch (C restatement, in place)."""
    fs = [np.ascontiguousarray(f, dtype=np.float64) for f in factors]
    dims = np.asarray(t.shape, dtype=np.int64)
    lib().oracle_ccd_sweep(t.order, _p(dims, _i64p), t.nnz, fs[0].shape[1],
                           _p(t.coords(), _i64p), _p(t.values, _f64p), _ptr_array(fs),
                           float(reg))
    for n in range(len(factors)):
        factors[n] = fs[n]


def sgd_sweep(t: OTensor, factors, reg: float, step: float, rate: float,
              seed: int, path: tuple):
    """optim.py:300-330 with the least-squares loss (losses.py:41-48)."""
    s = sample(t, rate, seed, path)
    shrink = 2.0 * step * reg * rate
    if s.nnz == 0:
        for mode in range(t.order):
            factors[mode] = factors[mode] - shrink * factors[mode]
        return
    model = tttp(s.with_values(np.ones(s.nnz)), factors)
    phi1 = s.with_values(2.0 * (model - s.values))
    grads = [mttkrp(phi1, factors, mode) for mode in range(t.order)]
    for mode in range(t.order):
        updated = factors[mode] - step * grads[mode] - shrink * factors[mode]
        if not np.isfinite(np.sum(updated)):
            raise OracleError("diverged", mode)
        factors[mode] = updated


def rmse(t: OTensor, factors) -> float:
    """losses.py:141-150."""
    model = tttp(t.with_values(np.ones(t.nnz)), factors)
    diff = t.values - model
    return float(np.sqrt(np.dot(diff, diff) / t.nnz))


def objective_ls(t: OTensor, factors, reg: float) -> float:
    """losses.py:126-138 with phi = (t - m)^2."""
    model = tttp(t.with_values(np.ones(t.nnz)), factors)
    total = float(np.sum((t.values - model) ** 2))
    if reg:
        total += reg * sum(float(np.sum(f * f)) for f in factors)
    return total


# ---------------------------------------------------------------------------
# second-order step (optim.py:334-598), restated on the oracle kernels.
# Losses are given as (dphi, d2phi) callables of (t, m) (losses.py:41-104).

def loss_derivs(ident: str):
    """losses.py:41-79: least squares and Poisson log link (m clamped at 50)."""
    if ident == "ls":
        return (lambda tv, m: 2.0 * (m - tv),
                lambda tv, m: np.full_like(np.asarray(m, dtype=np.float64), 2.0))
    if ident == "poisson":
        def ex(m):
            return np.exp(np.minimum(np.asarray(m, dtype=np.float64), 50.0))
        return (lambda tv, m: ex(m) - tv, lambda tv, m: ex(m))
    raise OracleError("loss", ident)


def gradient_blocks(t: OTensor, factors, ident: str, reg: float):
    """optim.py:336-345."""
    dphi, _ = loss_derivs(ident)
    model = tttp(t.with_values(np.ones(t.nnz)), factors)
    phi1 = t.with_values(dphi(t.values, model))
    return [mttkrp(phi1, factors, d) + 2.0 * reg * factors[d] for d in range(t.order)]


def hessian_matvec(phi1: OTensor, phi2: OTensor, factors, x_blocks, variant: str,
                   reg: float):
    """optim.py:348-384 (composed form: N substituted TTTPs, one MTTKRP per mode,
    Newton cross terms as MTTKRPs of phi1 with one substituted slot)."""
    n = len(factors)
    z = np.zeros(phi2.nnz)
    for p in range(n):
        sub = list(factors)
        sub[p] = x_blocks[p]
        z += tttp(phi2, sub)
    zt = phi2.with_values(z)
    y = [mttkrp(zt, factors, d) + 2.0 * reg * x_blocks[d] for d in range(n)]
    if variant == "newton":
        for d in range(n):
            for p in range(n):
                if p != d:
                    sub = list(factors)
                    sub[p] = x_blocks[p]
                    y[d] += mttkrp(phi1, sub, d)
    return y


def _bdot(a, b) -> float:
    return float(sum(np.sum(x * y) for x, y in zip(a, b)))


def pcg(matvec, precond, rhs, rel_tol: float, max_iters: int):
    """optim.py:492-531."""
    x = [np.zeros_like(b) for b in rhs]
    r = [b.copy() for b in rhs]
    b_norm = math.sqrt(_bdot(rhs, rhs))
    if b_norm == 0.0:
        return x, 0
    z = precond(r)
    p = [zi.copy() for zi in z]
    rz = _bdot(r, z)
    for it in range(1, max_iters + 1):
        ap = matvec(p)
        p_ap = _bdot(p, ap)
        if not math.isfinite(p_ap):
            raise OracleError("cg_curvature")
        if p_ap <= 0.0:
            return x, it - 1
        alpha = rz / p_ap
        for d in range(len(x)):
            x[d] += alpha * p[d]
            r[d] -= alpha * ap[d]
        res = math.sqrt(_bdot(r, r))
        if res / b_norm < rel_tol:
            return x, it
        z = precond(r)
        rz_new = _bdot(r, z)
        beta = rz_new / rz
        rz = rz_new
        for d in range(len(p)):
            p[d] = z[d] + beta * p[d]
    return x, max_iters


def rebalance(factors) -> None:
    """optim.py:534-555."""
    norms = np.stack([np.linalg.norm(f, axis=0) for f in factors])
    ok = np.all(norms > 0.0, axis=0)
    if not np.any(ok):
        return
    target = np.exp(np.log(norms[:, ok]).mean(axis=0))
    for n in range(len(factors)):
        scale = np.ones(norms.shape[1])
        scale[ok] = target / norms[n, ok]
        factors[n] *= scale


def gn_step(t: OTensor, factors, ident: str, reg: float, cg_tol: float, cg_max: int,
            variant: str = "gauss_newton", damping_state: dict | None = None,
            gn_damping: float = 0.0, gn_damping_decay: float = 0.5) -> int:
    """optim.py:558-598 (in place); returns the CG iterations used."""
    dphi, d2phi = loss_derivs(ident)
    model = tttp(t.with_values(np.ones(t.nnz)), factors)
    phi1 = t.with_values(dphi(t.values, model))
    phi2 = t.with_values(d2phi(t.values, model))
    if np.any(phi2.values < 0.0):
        raise OracleError("negative_curvature")
    n = t.order
    grad = [mttkrp(phi1, factors, d) + 2.0 * reg * factors[d] for d in range(n)]
    grams = [gram_blocks(phi2, factors, d) for d in range(n)]
    st = damping_state if damping_state is not None else {}
    if gn_damping > 0.0 and st.get("d") is None:
        st["d"] = gn_damping * float(np.mean([np.mean(np.diagonal(g, axis1=1, axis2=2))
                                              for g in grams]))
    reg_eff = reg + (st.get("d") or 0.0)
    eye = np.eye(factors[0].shape[1])
    systems = [g + 2.0 * reg_eff * eye for g in grams]

    def precond(blocks):
        return [np.linalg.solve(a, b[:, :, None])[:, :, 0] for a, b in zip(systems, blocks)]

    def matvec(x):
        return hessian_matvec(phi1, phi2, factors, x, variant, reg_eff)

    delta, used = pcg(matvec, precond, [-g for g in grad], cg_tol, cg_max)
    for d in range(n):
        factors[d] = factors[d] + delta[d]
    rebalance(factors)
    if st.get("d") is not None:
        st["d"] *= gn_damping_decay
    return used
