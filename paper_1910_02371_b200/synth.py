"""Seeded synthetic inputs for the BASELINE.json configurations.

The reference measures on the Netflix tensor and on random tensors; neither is
available here, so every input is synthesised on the host with a seeded numpy
``Generator`` following SURVEY.md section 8(d) (shapes, nnz, value laws only --
no dataset content).  CPU oracle and GPU path consume identical bytes.

Returned tensors are ``(shape, keys uint64 sorted, values f64)`` triples plus
factor lists, i.e. exactly what ``SparseTensor(shape, keys, values)``
(reference ``core.py:115``) accepts.
"""

from __future__ import annotations

import numpy as np

CFG1_SEED = 1
CFG2_SEED = 2
CFG3_SEED = 3
CFG4_SEED = 4
CFG5_SEED = 5


def _delinearize(keys, dims):
    rem = keys.copy()
    coords = [None] * len(dims)
    for n in range(len(dims) - 1, -1, -1):
        d = np.uint64(dims[n])
        coords[n] = (rem % d).astype(np.int64)
        rem //= d
    return coords


def _model_values(factors, coords):
    out = np.zeros(coords[0].size)
    rank = factors[0].shape[1]
    for lo in range(0, rank, 32):
        hi = min(lo + 32, rank)
        prod = factors[0][coords[0], lo:hi].copy()
        for n in range(1, len(factors)):
            prod *= factors[n][coords[n], lo:hi]
        out += prod.sum(axis=1)
    return out


def distinct_uniform_keys(rng, space: int, m: int) -> np.ndarray:
    """m distinct keys uniform on [0, space), sorted (draw, unique, top up,
    then a uniform random subset of exactly m -- never a lowest-k truncation,
    cf. the bias noted for cli._random_tensor in SURVEY.md 3.5)."""
    if m > space:
        raise ValueError("more keys than cells")
    if space <= 4 * m:
        keys = rng.choice(space, m, replace=False)
        return np.sort(keys).astype(np.uint64)
    keys = np.unique(rng.integers(0, space, size=int(m * 1.001) + 16, dtype=np.uint64))
    while keys.size < m:
        extra = rng.integers(0, space, size=(m - keys.size) * 2 + 16, dtype=np.uint64)
        keys = np.unique(np.concatenate([keys, extra]))
    if keys.size > m:
        pick = np.sort(rng.permutation(keys.size)[:m])
        keys = keys[pick]
    return keys


def cfg1(seed: int = CFG1_SEED):
    """BASELINE cfg 1: 200^3, 80,000 uniform distinct nonzeros, values =
    rank-5 U(0,1) CP model + N(0, sigma=0.01) noise; R=10 factors U(0,1)."""
    rng = np.random.default_rng(seed)
    shape = (200, 200, 200)
    keys = distinct_uniform_keys(rng, 200 ** 3, 80_000)
    truth = [rng.random((d, 5)) for d in shape]
    coords = _delinearize(keys, shape)
    values = _model_values(truth, coords) + rng.normal(0.0, 0.01, keys.size)
    factors = [rng.random((d, 10)) for d in shape]
    return shape, keys, values, factors


def cfg2(seed: int = CFG2_SEED, nnz: int = 10_000_000, rank: int = 16):
    """BASELINE cfg 2: 10^4 x 10^4 x 10^4, 1e7 uniform distinct nonzeros,
    values N(0,1), R=16 factors N(0, 1/R)."""
    rng = np.random.default_rng(seed)
    shape = (10_000, 10_000, 10_000)
    keys = distinct_uniform_keys(rng, 10 ** 12, nnz)
    values = rng.standard_normal(keys.size)
    factors = [rng.standard_normal((d, rank)) * np.sqrt(1.0 / rank) for d in shape]
    return shape, keys, values, factors


def cfg2_shard(rank: int, world: int, seed: int = CFG2_SEED, nnz: int = 10_000_000,
               R: int = 16):
    """Weak-scaling shard ``rank`` of a (world x nnz)-nonzero tensor over the
    cfg 2 index space: the shard holds nnz distinct uniform keys of the
    rank's contiguous slice of [0, 10^12), so the union over ranks is one
    sorted tensor partitioned into contiguous nonzero ranges (SURVEY.md 8(e)
    nnz sharding).  Factors are replicated (one draw for every rank).
    world == 1 is exactly ``cfg2``."""
    if world == 1:
        return cfg2(seed, nnz, R)
    space = 10 ** 12
    lo, hi = space * rank // world, space * (rank + 1) // world
    rng = np.random.default_rng([seed, rank, world])
    keys = np.uint64(lo) + distinct_uniform_keys(rng, hi - lo, nnz)
    values = rng.standard_normal(keys.size)
    frng = np.random.default_rng([seed, 99])
    shape = (10_000, 10_000, 10_000)
    factors = [frng.standard_normal((d, R)) * np.sqrt(1.0 / R) for d in shape]
    return shape, keys, values, factors


def zipf_indices(rng, dim: int, size: int, alpha: float = 1.0) -> np.ndarray:
    """Bounded Zipf(alpha) over 0..dim-1 by inverse CDF on weights 1/k^alpha."""
    w = 1.0 / np.arange(1, dim + 1, dtype=np.float64) ** alpha
    cdf = np.cumsum(w)
    cdf /= cdf[-1]
    u = rng.random(size)
    return np.minimum(np.searchsorted(cdf, u, side="right"), dim - 1).astype(np.int64)


def cfg3(seed: int = CFG3_SEED, nnz: int = 100_480_507,
         shape=(480_189, 17_770, 2_182)):
    """BASELINE cfg 3 stand-in (shape and nnz of the paper's Netflix run only):
    modes 0, 1 bounded Zipf(1), mode 2 uniform, distinct coordinates (dedupe
    and top up), a uniform subset of exactly nnz, values uniform {1..5}."""
    rng = np.random.default_rng(seed)
    shape = tuple(int(d) for d in shape)
    keys = np.empty(0, dtype=np.uint64)
    draws = int(nnz * 1.05)
    while keys.size < nnz:
        i0 = zipf_indices(rng, shape[0], draws).astype(np.uint64)
        i1 = zipf_indices(rng, shape[1], draws).astype(np.uint64)
        i2 = rng.integers(0, shape[2], draws, dtype=np.uint64)
        k = (i0 * np.uint64(shape[1]) + i1) * np.uint64(shape[2]) + i2
        keys = np.unique(np.concatenate([keys, k]))
        draws = max(int((nnz - keys.size) * 1.5), 1024)
    if keys.size > nnz:
        keys = keys[np.sort(rng.permutation(keys.size)[:nnz])]
    values = rng.integers(1, 6, keys.size).astype(np.float64)
    return shape, keys, values


def cfg4(seed: int = CFG4_SEED, n: int = 800, rank: int = 64):
    """BASELINE cfg 4: dense n^3 N(0,1) tensor, R=64 factors N(0,1)."""
    rng = np.random.default_rng(seed)
    x = rng.standard_normal((n, n, n))
    factors = [rng.standard_normal((n, rank)) for _ in range(3)]
    return x, factors


def cfg5(seed: int = CFG5_SEED, nnz: int = 1_000_000_000,
         shape=(100_000, 100_000, 100_000, 1_000), rank: int = 64):
    """BASELINE cfg 5: order 4, uniform distinct keys, values = rank-8 CP model
    (truth factors N(0, 1/8)) + N(0, 0.1) noise, fp32; R=64 factors."""
    rng = np.random.default_rng(seed)
    shape = tuple(int(d) for d in shape)
    space = int(np.prod(np.array(shape, dtype=object)))
    keys = distinct_uniform_keys(rng, space, nnz)
    truth = [rng.standard_normal((d, 8)) * np.sqrt(1.0 / 8) for d in shape]
    coords = _delinearize(keys, shape)
    values = (_model_values(truth, coords) + rng.normal(0.0, 0.1, keys.size))
    factors = [(rng.standard_normal((d, rank)) * np.sqrt(1.0 / rank)) for d in shape]
    return shape, keys, values.astype(np.float32), [f.astype(np.float32) for f in factors]


def cfg3_device(seed: int = CFG3_SEED, nnz: int = 100_480_507,
                shape=(480_189, 17_770, 2_182), device="cuda"):
    """cfg 3 synthesised on the GPU (torch RNG, same laws as ``cfg3``):
    returns (shape, sorted int64 keys on device, f64 values on device).
    Seconds instead of minutes at full size; deterministic for a given seed
    and GPU type.  Used by the ALS / CCD++ benchmarks."""
    import torch
    shape = tuple(int(d) for d in shape)
    g = torch.Generator(device=device)
    g.manual_seed(int(seed))

    def zipf(dim, size):
        w = 1.0 / torch.arange(1, dim + 1, dtype=torch.float64, device=device)
        cdf = torch.cumsum(w, 0)
        cdf /= cdf[-1].clone()
        u = torch.rand(size, generator=g, dtype=torch.float64, device=device)
        return torch.clamp(torch.searchsorted(cdf, u, right=True), max=dim - 1)

    keys = torch.empty(0, dtype=torch.int64, device=device)
    draws = int(nnz * 1.05)
    while keys.numel() < nnz:
        i0 = zipf(shape[0], draws)
        i1 = zipf(shape[1], draws)
        i2 = torch.randint(0, shape[2], (draws,), generator=g, device=device)
        k = (i0 * shape[1] + i1) * shape[2] + i2
        del i0, i1, i2
        keys = torch.unique(torch.cat([keys, k]))
        del k
        draws = max(int((nnz - keys.numel()) * 1.5), 1024)
    if keys.numel() > nnz:
        pick = torch.randperm(keys.numel(), generator=g, device=device)[:nnz]
        keys = keys[torch.sort(pick).values]
    values = torch.randint(1, 6, (nnz,), generator=g, device=device).to(torch.float64)
    return shape, keys, values


def cfg5_device(seed: int = CFG5_SEED, nnz: int = 1_000_000_000,
                shape=(100_000, 100_000, 100_000, 1_000), rank: int = 64, device="cuda",
                with_keys: bool = False):
    """BASELINE cfg 5 synthesised on the GPU: order 4, nnz distinct uniform
    keys, values = rank-8 CP model (truth factors N(0, 1/8), evaluated with
    the library's own TTTP kernel) + N(0, 0.1) noise, fp32; R=64 factors
    N(0, 1/R).  Returns (shape, tensor, f32 values, f32 factors) and, with
    ``with_keys``, the sorted int64 device keys as a fifth item."""
    import torch
    shape = tuple(int(d) for d in shape)
    space = 1
    for d in shape:
        space *= d
    g = torch.Generator(device=device)
    g.manual_seed(int(seed))
    keys = torch.unique(torch.randint(0, space, (int(nnz * 1.0001) + 64,), generator=g,
                                      device=device, dtype=torch.int64))
    while keys.numel() < nnz:
        extra = torch.randint(0, space, (2 * (nnz - keys.numel()) + 64,), generator=g,
                              device=device, dtype=torch.int64)
        keys = torch.unique(torch.cat([keys, extra]))
    if keys.numel() > nnz:
        pick = torch.randperm(keys.numel(), generator=g, device=device)[:nnz]
        keys = keys[torch.sort(pick).values]
    truth = [torch.randn((d, 8), generator=g, device=device) * (1.0 / 8) ** 0.5 for d in shape]
    noise = torch.randn((nnz,), generator=g, device=device) * 0.1
    factors = [torch.randn((d, rank), generator=g, device=device) * (1.0 / rank) ** 0.5
               for d in shape]
    from .core import SparseTensor
    from .losses import tttp_affine
    t = SparseTensor.from_device(shape, keys, noise)
    values = tttp_affine(t, truth, 1.0, 1.0, torch.float32)  # model + noise
    if with_keys:
        return shape, t, values, factors, keys
    return shape, t, values, factors
