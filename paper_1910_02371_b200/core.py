"""Sparse tensors with a device-resident sparsity pattern.

Same public surface as the reference's core.py (``SparseTensor``,
``RngState``, ``linearize[_many]``, ``delinearize[_many]``, ``from_coords``,
``build_tensor``, ``counting_sort_by_mode``, ``model_values``,
``gen_low_rank``), re-designed around the B200: the first kernel call on a
tensor uploads its sorted uint64 keys once and builds a *device pattern*
(``libcpfit_b200``: int32 coordinates per mode, delinearized on the GPU),
and every mode grouping (stable radix sort, segment offsets, work tasks) is
built on the device on first use and cached in that pattern.  Tensors made
with ``with_values`` share the pattern exactly like the reference shares its
``_coords`` / ``_groups`` caches (core.py:159-167), so ALS/CCD/SGD sweeps
never re-sort.  Values live on the device per dtype; host ``keys`` /
``values`` are materialised lazily for device-born tensors (samples, kernel
outputs).

Ingest (``from_coords`` / ``build_tensor``: linearize, stable sort,
duplicate merge) runs on the device too; only scalar helpers (linearize on a
tuple) and the seeded synthetic generators stay on the host.
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .exceptions import DataError
from .validation import _is_torch, check_mode, check_shape

DEFAULT_CELL_CAP = 1 << 26


# ---------------------------------------------------------------------------
# device plumbing (torch = device memory + streams)

def _torch():
    import torch
    return torch


_DEVICES: dict = {}
_CUDA_OK = None


def cuda_device():
    """torch.device of the current CUDA device (cached per index: the API
    entry points call this many times per call)."""
    global _CUDA_OK
    torch = _torch()
    if _CUDA_OK is None:
        _CUDA_OK = torch.cuda.is_available()
    if not _CUDA_OK:
        raise RuntimeError("cpfit-b200 kernels need a CUDA device (B200, sm_100a); "
                           "there is no CPU fallback")
    idx = torch._C._cuda_getDevice()
    dev = _DEVICES.get(idx)
    if dev is None:
        dev = _DEVICES[idx] = torch.device("cuda", idx)
    return dev


def current_stream() -> int:
    """Raw cudaStream_t of torch's current stream on the current device (the
    library launches on it)."""
    torch = _torch()
    try:
        return torch._C._cuda_getCurrentRawStream(torch._C._cuda_getDevice())
    except AttributeError:  # older torch
        return torch.cuda.current_stream().cuda_stream


def to_host_sm(t) -> np.ndarray:
    """Small device tensor -> numpy with the copy done by a kernel writing
    pinned host memory (cpfit_copy_to_host): it does not queue behind a large
    device->host DMA still draining on the copy engine."""
    torch = _torch()
    h = torch.empty(tuple(t.shape), dtype=t.dtype, pin_memory=True)
    t = t.contiguous()
    _lib.check(_lib.load().cpfit_copy_to_host(
        t.numel() * t.element_size(), ctypes.c_void_p(t.data_ptr()),
        ctypes.c_void_p(h.data_ptr()), ctypes.c_void_p(current_stream())), "copy_to_host")
    torch.cuda.current_stream().synchronize()
    return h.numpy()


def to_host(t, dtype=None) -> np.ndarray:
    """Device tensor -> numpy through torch's pinned host cache: the copy is a
    direct DMA at full PCIe rate, and the pinned block goes back to torch's
    cache when the returned array is released."""
    torch = _torch()
    if dtype is not None and t.dtype != dtype:
        t = t.to(dtype)
    h = torch.empty(tuple(t.shape), dtype=t.dtype, pin_memory=True)
    h.copy_(t)
    return h.numpy()


class _CudaArray:
    """Zero-copy __cuda_array_interface__ view of library-owned device memory."""

    def __init__(self, ptr: int, n: int, typestr: str):
        self.__cuda_array_interface__ = {
            "shape": (int(n),), "typestr": typestr, "data": (int(ptr), False),
            "version": 3, "strides": None, "stream": None,
        }


def device_view(ptr: int, n: int, typestr: str, owner=None):
    """torch view of library-owned memory (keep ``owner`` alive while used)."""
    torch = _torch()
    arr = _CudaArray(ptr, n, typestr)
    # torch keeps the interface object alive as long as the tensor: hanging
    # the owner on it ties the pattern's lifetime to every view of its memory
    arr._owner = owner
    return torch.as_tensor(arr, device=cuda_device())


class DevicePattern:
    """Owner of one ``cpfit_pattern`` handle (device coords + cached layouts)."""

    def __init__(self, shape, nnz: int, handle: int, task_size: int | None = None):
        self.shape = tuple(shape)
        self.nnz = int(nnz)
        self._h = ctypes.c_void_p(handle)
        self._stream = None      # the one stream every call so far was issued on
        self._streams_mixed = False
        if task_size is not None:
            _lib.check(_lib.load().cpfit_pattern_set_task_size(self.handle, int(task_size)))

    @property
    def handle(self):
        """The C handle.  Every use goes through here, so the pattern knows
        whether all of its device work was issued on a single stream (then it
        can be released stream-ordered, without a device synchronisation)."""
        h = self._h
        if h is not None:
            s = current_stream()
            if self._stream is None:
                self._stream = s
            elif self._stream != s:
                self._streams_mixed = True
        return h

    @classmethod
    def from_keys(cls, shape, keys):
        """Upload sorted uint64 keys (numpy or CUDA tensor) and delinearize."""
        torch = _torch()
        dev = cuda_device()
        if isinstance(keys, np.ndarray):
            k = torch.from_numpy(np.ascontiguousarray(keys, dtype=np.uint64).view(np.int64))
            k = k.to(dev, non_blocking=False)
        else:
            k = keys.to(dev).view(torch.int64).contiguous()
        dims = (ctypes.c_int64 * len(shape))(*shape)
        out = ctypes.c_void_p()
        _lib.check(_lib.load().cpfit_pattern_create(
            len(shape), dims, int(k.numel()), ctypes.c_void_p(k.data_ptr()),
            ctypes.c_void_p(current_stream()), ctypes.byref(out)), "pattern_create")
        # keys are consumed by the delinearize kernel on the current stream;
        # keep them alive until it has run
        _torch().cuda.current_stream().synchronize()
        return cls(shape, int(k.numel()), out.value)

    @classmethod
    def from_device_coords(cls, shape, coords):
        """Pattern from per-mode int32 CUDA coordinate tensors (canonical order)."""
        n = int(coords[0].numel()) if coords else 0
        dims = (ctypes.c_int64 * len(shape))(*shape)
        arr = _lib.ptr_array([c.data_ptr() for c in coords])
        out = ctypes.c_void_p()
        _lib.check(_lib.load().cpfit_pattern_create_coords(
            len(shape), dims, n, arr, ctypes.c_void_p(current_stream()),
            ctypes.byref(out)), "pattern_create_coords")
        _torch().cuda.current_stream().synchronize()
        return cls(shape, n, out.value)

    def coords(self, mode: int):
        p = ctypes.c_void_p()
        _lib.check(_lib.load().cpfit_pattern_coords(self.handle, int(mode), ctypes.byref(p)))
        return device_view(p.value, self.nnz, "<i4", self)

    def mode_group(self, mode: int):
        perm = ctypes.c_void_p()
        offs = ctypes.c_void_p()
        _lib.check(_lib.load().cpfit_pattern_mode_group(
            self.handle, int(mode), ctypes.c_void_p(current_stream()), ctypes.byref(perm),
            ctypes.byref(offs)), "mode_group")
        return (device_view(perm.value, self.nnz, "<i4", self),
                device_view(offs.value, self.shape[mode] + 1, "<i8", self))

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value and _lib._lib is not None:
            try:
                if self._stream is not None and not self._streams_mixed:
                    _lib.load().cpfit_pattern_destroy_async(h, ctypes.c_void_p(self._stream))
                else:
                    _lib.load().cpfit_pattern_destroy(h)
            except Exception:  # interpreter shutdown
                pass
            self._h = None


@dataclass
class _Shared:
    """Pattern-level caches shared through ``with_values`` (core.py:159-167)."""

    coords: tuple | None = None          # host int64 coords (on request)
    groups: dict = field(default_factory=dict)  # host (perm, offsets) per mode
    pattern: DevicePattern | None = None
    task_size: int | None = None
    parent: object = None                # sampled patterns: positions in the source


def _dtype_code(dtype) -> int:
    torch = _torch()
    if dtype == torch.float64:
        return _lib.F64
    if dtype == torch.float32:
        return _lib.F32
    raise ValueError(f"unsupported dtype {dtype}")


# ---------------------------------------------------------------------------
# RNG (core.py:25-46)

@dataclass(frozen=True)
class RngState:
    """Splittable counter-based stream: numpy Philox4x64-10 keyed by
    SeedSequence(seed, spawn_key=path), identical to the reference."""

    seed: int
    path: tuple[int, ...] = field(default=())
    algorithm: str = "philox"

    def generator(self) -> np.random.Generator:
        ss = np.random.SeedSequence(entropy=self.seed, spawn_key=self.path)
        return np.random.Generator(np.random.Philox(ss))

    def child(self, key: int) -> "RngState":
        return RngState(self.seed, self.path + (int(key),), self.algorithm)

    def split(self, n: int) -> list["RngState"]:
        return [self.child(i) for i in range(n)]

    def philox_key(self) -> tuple[int, int]:
        """The 2x64-bit Philox key (what the device sampler consumes)."""
        ss = np.random.SeedSequence(entropy=self.seed, spawn_key=self.path)
        key = np.random.Philox(ss).state["state"]["key"]
        return int(key[0]), int(key[1])


# ---------------------------------------------------------------------------
# index arithmetic (core.py:49-102; host utilities)

def linearize(coords, dims) -> int:
    """Row-major key of one coordinate tuple (last mode fastest)."""
    dims = check_shape(dims)
    if len(coords) != len(dims):
        raise ValueError(f"expected {len(dims)} coordinates, got {len(coords)}")
    key = 0
    for n, extent in enumerate(dims):
        c = int(coords[n])
        if c < 0 or c >= extent:
            raise ValueError(f"coordinate {c} out of range [0, {extent}) in mode {n}")
        key = key * extent + c          # Horner in mixed radix
    return key


def delinearize(key: int, dims) -> tuple[int, ...]:
    dims = check_shape(dims)
    rest = int(key)
    if rest < 0 or rest >= math.prod(dims):
        raise ValueError(f"key {rest} out of range for shape {dims}")
    digits = []
    for extent in reversed(dims):
        rest, digit = divmod(rest, extent)
        digits.append(digit)
    return tuple(reversed(digits))


def linearize_many(coord_arrays, dims) -> np.ndarray:
    """Vectorised ``linearize`` (host; the device ingest is cpfit_from_coords)."""
    dims = check_shape(dims)
    if len(coord_arrays) != len(dims):
        raise ValueError("one coordinate array per mode required")
    keys = np.zeros(len(coord_arrays[0]) if len(coord_arrays) else 0, dtype=np.uint64)
    for n, extent in enumerate(dims):
        col = np.asarray(coord_arrays[n])
        if col.size and (col.min() < 0 or col.max() >= extent):
            raise ValueError(f"coordinate out of range [0, {extent}) in mode {n}")
        keys *= np.uint64(extent)
        keys += col.astype(np.uint64)
    return keys


def delinearize_many(keys, dims) -> tuple[np.ndarray, ...]:
    dims = check_shape(dims)
    rest = np.array(keys, dtype=np.uint64)        # private copy, consumed below
    out: list = []
    for extent in reversed(dims):
        rest, digit = np.divmod(rest, np.uint64(extent))
        out.append(digit.astype(np.int64))
    return tuple(reversed(out))


# ---------------------------------------------------------------------------
# SparseTensor

class SparseTensor:
    """Order-N sparse tensor in sorted linearized-key coordinate format.

    Invariants (core.py:105-131): keys strictly increasing uint64, every key
    < prod(dims), len(keys) == len(values); explicit zeros are retained.
    """

    __slots__ = ("shape", "_keys", "_values", "_shared", "_dvals", "_sorted",
                 "_keys_fn", "_nnz", "_pending", "__weakref__")

    def __init__(self, shape, keys, values, validate: bool = True):
        shape = check_shape(shape)
        keys = np.ascontiguousarray(keys, dtype=np.uint64)
        values = np.ascontiguousarray(values, dtype=np.float64)
        if validate:
            if keys.ndim != 1 or values.ndim != 1 or keys.shape != values.shape:
                raise ValueError("keys and values must be 1-D of equal length")
            if keys.size:
                if np.any(keys[1:] <= keys[:-1]):
                    raise ValueError("keys must be strictly increasing")
                if int(keys[-1]) >= math.prod(shape):
                    raise ValueError("key out of range for shape")
        self.shape = shape
        self._keys = keys
        self._values = values
        self._nnz = int(keys.size)
        self._shared = _Shared()
        self._dvals = {}
        self._sorted = {}
        self._keys_fn = None
        self._pending = None

    # -- construction of device-born tensors --------------------------------
    @classmethod
    def _device_born(cls, shape, nnz, shared, dvalues, keys_fn=None, host_values=None):
        t = cls.__new__(cls)
        t.shape = tuple(shape)
        t._keys = None
        t._values = host_values
        t._nnz = int(nnz)
        t._shared = shared
        t._dvals = {} if dvalues is None else {dvalues.dtype: dvalues}
        t._sorted = {}
        t._keys_fn = keys_fn
        t._pending = None
        return t

    @classmethod
    def from_device(cls, shape, keys, values) -> "SparseTensor":
        """Tensor whose sorted keys (int64/uint64 CUDA tensor) and values live
        on the device already: the pattern is built straight from them and
        host copies materialise only if ``keys`` / ``values`` are read."""
        shape = check_shape(shape)
        if keys.numel() != values.numel():
            raise ValueError("keys and values must be 1-D of equal length")
        shared = _Shared(pattern=DevicePattern.from_keys(shape, keys))
        host = {}

        def keys_fn():
            if "k" not in host:
                host["k"] = keys.cpu().numpy().view(np.uint64)
            return host["k"]
        return cls._device_born(shape, keys.numel(), shared, values.contiguous(),
                                keys_fn=keys_fn)

    @property
    def keys(self) -> np.ndarray:
        if self._keys is None:
            self._keys = np.ascontiguousarray(self._keys_fn(), dtype=np.uint64)
        return self._keys

    @property
    def values(self) -> np.ndarray:
        if self._values is None and self._pending is not None:
            # host values still streaming back (kernels.tttp numpy path)
            self._values = self._pending()
            self._pending = None
        if self._values is None:
            torch = _torch()
            dv = self._dvals.get(torch.float64)
            if dv is None:
                dv = next(iter(self._dvals.values()))
            self._values = to_host(dv, torch.float64)
        return self._values

    @property
    def order(self) -> int:
        return len(self.shape)

    @property
    def nnz(self) -> int:
        return self._nnz

    # -- device side ----------------------------------------------------------
    def device_pattern(self) -> DevicePattern:
        sh = self._shared
        if sh.pattern is None:
            sh.pattern = DevicePattern.from_keys(self.shape, self.keys)
            if sh.task_size is not None:
                _lib.check(_lib.load().cpfit_pattern_set_task_size(sh.pattern.handle,
                                                                  int(sh.task_size)))
        return sh.pattern

    def set_task_size(self, entries: int) -> None:
        """Entries per segmented-work task (before the first mode grouping)."""
        self._shared.task_size = int(entries)
        if self._shared.pattern is not None:
            _lib.check(_lib.load().cpfit_pattern_set_task_size(
                self._shared.pattern.handle, int(entries)))

    def device_values(self, dtype=None):
        """Values on the device in canonical (key) order, cached per dtype."""
        torch = _torch()
        dtype = dtype or torch.float64
        dv = self._dvals.get(dtype)
        if dv is None:
            src = next(iter(self._dvals.values()), None)
            if src is not None:
                dv = src.to(dtype)
            else:
                dv = torch.from_numpy(self.values).to(cuda_device()).to(dtype)
            self._dvals[dtype] = dv
        return dv

    def sorted_values(self, mode: int, dtype=None):
        """Values permuted into the mode-sorted order of ``mode`` (cached)."""
        torch = _torch()
        dtype = dtype or torch.float64
        key = (int(mode), dtype)
        sv = self._sorted.get(key)
        if sv is None:
            src = self.device_values(dtype)
            sv = torch.empty_like(src)
            _lib.check(_lib.load().cpfit_permute_values(
                self.device_pattern().handle, int(mode), _dtype_code(dtype),
                ctypes.c_void_p(src.data_ptr()), ctypes.c_void_p(sv.data_ptr()),
                ctypes.c_void_p(current_stream())), "permute_values")
            self._sorted[key] = sv
        return sv

    # -- reference API --------------------------------------------------------
    def coords(self) -> tuple[np.ndarray, ...]:
        """Per-mode int64 coordinates (device delinearize, cached)."""
        sh = self._shared
        if sh.coords is None:
            if self.nnz == 0:
                sh.coords = tuple(np.zeros(0, dtype=np.int64) for _ in self.shape)
            else:
                pat = self.device_pattern()
                sh.coords = tuple(pat.coords(n).cpu().numpy().astype(np.int64)
                                  for n in range(self.order))
        return sh.coords

    def mode_group(self, mode: int):
        """Cached (perm, offsets) grouping by mode index (device radix sort;
        bit-exact with counting_sort_by_mode, core.py:234-249)."""
        mode = check_mode(mode, self.order)
        hit = self._shared.groups.get(mode)
        if hit is None:
            if self.nnz == 0:
                hit = (np.zeros(0, dtype=np.int64),
                       np.zeros(self.shape[mode] + 1, dtype=np.int64))
            else:
                perm, offs = self.device_pattern().mode_group(mode)
                hit = (perm.cpu().numpy().astype(np.int64), offs.cpu().numpy().copy())
            self._shared.groups[mode] = hit
        return hit

    def with_values(self, values) -> "SparseTensor":
        """New tensor sharing this pattern (and its device layouts)."""
        if type(values).__module__.startswith("torch"):
            if tuple(values.shape) != (self.nnz,):
                raise ValueError("values length must match nnz")
            return SparseTensor._device_born(
                self.shape, self.nnz, self._shared, values.contiguous(),
                keys_fn=lambda: self.keys)
        values = np.ascontiguousarray(values, dtype=np.float64)
        if values.shape != (self.nnz,):
            raise ValueError("values length must match nnz")
        out = SparseTensor._device_born(self.shape, self.nnz, self._shared, None,
                                        keys_fn=lambda: self.keys, host_values=values)
        if self._keys is not None:
            out._keys = self._keys
        return out

    def observation_mask(self) -> "SparseTensor":
        """Unit-valued tensor on the same pattern (core.py:169-171)."""
        if self._values is None and self._dvals:
            torch = _torch()
            return self.with_values(torch.ones(self.nnz, dtype=torch.float64,
                                               device=cuda_device()))
        return self.with_values(np.ones(self.nnz))

    def sample(self, rate: float, rng: RngState) -> "SparseTensor":
        """Keep each entry independently with probability ``rate`` (device
        Philox4x64-10, bit-exact with the reference's core.py:173-183)."""
        from .sampling import sample_tensor
        return sample_tensor(self, rate, rng)

    def norm_sq(self) -> float:
        return float(np.dot(self.values, self.values))

    def __repr__(self) -> str:
        return f"SparseTensor(shape={self.shape}, nnz={self.nnz})"


def build_tensor(entries, shape) -> SparseTensor:
    """core.py:192-205: unsorted ((coords...), value) pairs, duplicates summed
    -- through the device ingest like from_coords."""
    shape = check_shape(shape)
    if not entries:
        return SparseTensor(shape, np.empty(0, np.uint64), np.empty(0))
    for c, _ in entries:  # per-entry validation with the reference's messages
        linearize(c, shape)
    cols = np.array([tuple(c) for c, _ in entries], dtype=np.int64).reshape(len(entries), -1)
    values = np.fromiter((v for _, v in entries), dtype=np.float64, count=len(entries))
    return from_coords_device([cols[:, n] for n in range(len(shape))], values, shape)


def from_coords(coord_arrays, values, shape) -> SparseTensor:
    """core.py:208-218: per-mode coordinate arrays, duplicates summed.

    The whole ingest runs on the device (cpfit_from_coords: linearize, stable
    radix sort, duplicate merge in numpy's reduceat order; bit-identical keys
    and values); numpy inputs are uploaded first.  No CPU path."""
    shape = check_shape(shape)
    if len(coord_arrays) != len(shape):
        raise ValueError("one coordinate array per mode required")
    return from_coords_device(coord_arrays, values, shape)


def from_coords_device(coord_arrays, values, shape) -> SparseTensor:
    """from_coords on the device: coordinate arrays (int32 / int64, numpy or
    CUDA tensors, any order, duplicates allowed) and fp64 values -> a tensor
    whose sorted keys and merged values stay on the device."""
    torch = _torch()
    shape = check_shape(shape)
    if len(coord_arrays) != len(shape):
        raise ValueError("one coordinate array per mode required")
    dev = cuda_device()

    if _is_torch(values):
        vals = values.to(device=dev, dtype=torch.float64).contiguous().reshape(-1)
    else:
        vals = torch.from_numpy(np.ascontiguousarray(values, dtype=np.float64).reshape(-1)).to(dev)
    cs = []
    for q, c in enumerate(coord_arrays):
        if _is_torch(c):
            ct = c.to(dev)
            if ct.dtype not in (torch.int32, torch.int64):
                ct = ct.to(torch.int64)
        else:
            a = np.asarray(c)
            if a.dtype != np.int32:
                if a.size and a.dtype.kind == "u" and int(a.max()) > np.iinfo(np.int64).max:
                    raise ValueError(f"coordinate out of range [0, {shape[q]}) in mode {q}")
                a = a.astype(np.int64)
            ct = torch.from_numpy(np.ascontiguousarray(a)).to(dev)
        cs.append(ct.contiguous().reshape(-1))
    width = 4 if all(c.dtype == torch.int32 for c in cs) else 8
    if width == 8:
        cs = [c.to(torch.int64) for c in cs]
    n = int(vals.numel())
    if any(int(c.numel()) != n for c in cs):
        raise ValueError("coordinate arrays and values must have equal length")
    keys = torch.empty(n, dtype=torch.int64, device=dev)
    out = torch.empty(n, dtype=torch.float64, device=dev)
    nnz = ctypes.c_int64(0)
    bad = ctypes.c_int(-1)
    dims = (ctypes.c_int64 * len(shape))(*shape)
    arr = _lib.ptr_array([c.data_ptr() for c in cs])
    st = _lib.load().cpfit_from_coords(
        len(shape), dims, n, width, ctypes.cast(arr, ctypes.POINTER(ctypes.c_void_p)),
        ctypes.c_void_p(vals.data_ptr()), ctypes.c_void_p(keys.data_ptr()),
        ctypes.c_void_p(out.data_ptr()), ctypes.byref(nnz), ctypes.byref(bad),
        ctypes.c_void_p(current_stream()))
    if st != 0 and bad.value >= 0:
        raise ValueError(f"coordinate out of range [0, {shape[bad.value]}) in mode {bad.value}")
    _lib.check(st, "from_coords")
    m = nnz.value
    return SparseTensor.from_device(shape, keys[:m], out[:m])


def counting_sort_by_mode(t: SparseTensor, mode: int):
    """Stable grouping of entry positions by mode index -> (perm, offsets).

    Computed on the device (LSD radix sort, core.py:234-249 semantics)."""
    mode = check_mode(mode, t.order)
    return t.mode_group(mode)


def model_values(factors, coord_arrays, col_block: int = 32) -> np.ndarray:
    """Multilinear inner products sum_r prod_n A_n[i_n, r] at given coordinates.

    Host helper for the synthetic generators.  The summation order is the
    reference's (core.py:252-266: column blocks of ``col_block``, a row sum per
    block, blocks added left to right), so generated values are bit-identical."""
    mats = [np.asarray(f.cpu().numpy() if hasattr(f, "cpu") else f, dtype=np.float64)
            for f in factors]
    count = len(coord_arrays[0]) if len(coord_arrays) else 0
    total = np.zeros(count)
    rank = mats[0].shape[1]
    for first in range(0, rank, col_block):
        cols = slice(first, min(first + col_block, rank))
        block = mats[0][coord_arrays[0], cols].copy()
        for mat, idx in zip(mats[1:], coord_arrays[1:]):
            block *= mat[idx, cols]
        total += block.sum(axis=1)
    return total


def _observed_keys(shape, observed_fraction: float, g: np.random.Generator) -> np.ndarray:
    """Bernoulli(observed_fraction) mask over the enumerated cell space, as
    sorted keys (one uniform draw per cell, like the reference generators)."""
    cells = math.prod(shape)
    if observed_fraction >= 1.0:
        return np.arange(cells, dtype=np.uint64)
    return np.flatnonzero(g.random(cells) < observed_fraction).astype(np.uint64)


def _check_generator_args(shape, observed_fraction: float, cell_cap: int, hint: str):
    shape = check_shape(shape)
    if not 0.0 < observed_fraction <= 1.0:
        raise ValueError("observed_fraction must be in (0, 1]")
    cells = math.prod(shape)
    if cells > cell_cap:
        raise DataError(f"cell space {cells} exceeds enumeration cap {cell_cap}{hint}")
    return shape


_FACTOR_LAWS = {
    "uniform01": lambda g, size: g.random(size),
    "gaussian": lambda g, size: g.standard_normal(size),
}


def gen_low_rank(shape, rank: int, observed_fraction: float,
                 value_law: str = "uniform01", rng: RngState | None = None,
                 cell_cap: int = DEFAULT_CELL_CAP):
    """Random rank-``rank`` CP model observed on a Bernoulli mask -> (tensor,
    truth factors).  Draw order follows core.py:269-314 (factors mode by mode,
    then the mask), so a given RngState yields the reference's tensor."""
    shape = _check_generator_args(shape, observed_fraction, cell_cap,
                                  "; raise cell_cap explicitly for larger masks")
    g = (rng or RngState(0)).generator()
    truth = []
    for extent in shape:
        if value_law not in _FACTOR_LAWS:
            raise ValueError(f"unknown value_law {value_law!r}")
        truth.append(_FACTOR_LAWS[value_law](g, (extent, rank)))
    keys = _observed_keys(shape, observed_fraction, g)
    values = model_values(truth, delinearize_many(keys, shape))
    return SparseTensor(shape, keys, values, validate=False), truth


def _inverse_index_sum(coords) -> np.ndarray:
    # default test function of core.py:317-348: 1 / (1 + i_0 + i_1 + ...)
    acc = np.zeros(len(coords[0]))
    for c in coords:
        acc += c
    return 1.0 / (1.0 + acc)


def gen_function_tensor(shape, observed_fraction: float, rng: RngState | None = None,
                        func=None, cell_cap: int = DEFAULT_CELL_CAP) -> SparseTensor:
    """``func(coords)`` sampled on a Bernoulli mask (core.py:317-348)."""
    shape = _check_generator_args(shape, observed_fraction, cell_cap, "")
    keys = _observed_keys(shape, observed_fraction, (rng or RngState(0)).generator())
    evaluate = func or _inverse_index_sum
    return SparseTensor(shape, keys, evaluate(delinearize_many(keys, shape)), validate=False)
