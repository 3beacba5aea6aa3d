"""Multi-process (gloo, world size 2, CPU) tests of the sharding logic in
paper_1910_02371_b200.dist, with the CPU oracle as the row-local compute:
the row-sharded ALS sweep with an all-gather of factor rows must reproduce
the single-process sweep bit for bit; the nonzero-sharded SGD sample must be
the single-process sample bit for bit and the all-reduced gradients must
match within 1e-12; the nonzero-sharded CCD++ sweep and SGD steps must match
the single-process sweeps within 1e-10 / 1e-12 (the all-reduce reassociates
the per-row sums) with the replicas bit-identical."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import oracle as O
from paper_1910_02371_b200 import dist as D
from paper_1910_02371_b200 import synth


class OracleBackend:
    xp = np

    def make_shard(self, shape, keys, values):
        return O.OTensor(tuple(int(d) for d in shape), np.asarray(keys, dtype=np.uint64),
                         np.asarray(values, dtype=np.float64))

    def als_mode(self, shard, factors, mode, reg, lo, hi):
        fs = [None if n == mode else f for n, f in enumerate(factors)]
        rhs = O.mttkrp(shard, fs, mode)
        mask = shard.with_values(np.ones(shard.nnz))
        return O.solve_factor(mask, fs, rhs, mode, reg=reg)

    def to_comm(self, x):
        return torch.from_numpy(np.ascontiguousarray(x))

    def from_comm(self, x):
        return x.numpy().copy()

    def empty_comm(self, shape, like):
        return torch.empty(shape, dtype=like.dtype)

    def cat(self, parts):
        return torch.cat(parts, 0)

    # nonzero shards (ShardedCCD / ShardedSGD)
    def make_nnz_shard(self, shape, keys, values):
        return self.make_shard(shape, keys, values)

    def ccd_begin(self, shard, factors):
        model = O.tttp(shard.with_values(np.ones(shard.nnz)), factors)
        return {"cols": [np.ascontiguousarray(f.T) for f in factors],
                "resid": shard.values - model, "coords": shard.coords()}

    def ccd_numden(self, shard, st, r, mode):
        c = st["coords"]
        part = np.ones(shard.nnz)
        for q in range(shard.order):
            if q != mode:
                part = part * st["cols"][q][r][c[q]]
        rho = st["resid"] + part * st["cols"][mode][r][c[mode]]
        st["part"], st["rho"] = part, rho
        d = shard.shape[mode]
        return torch.from_numpy(np.concatenate([
            np.bincount(c[mode], weights=rho * part, minlength=d),
            np.bincount(c[mode], weights=part * part, minlength=d)]))

    def ccd_apply(self, shard, st, r, mode, nd, reg):
        d = shard.shape[mode]
        nd = nd.numpy()
        old = st["cols"][mode][r]
        dr = nd[d:] + reg
        new = np.where(dr > 0.0, nd[:d] / np.where(dr > 0.0, dr, 1.0), old)
        st["resid"] = st["rho"] - st["part"] * new[st["coords"][mode]]
        st["cols"][mode][r] = new

    def ccd_end(self, st, factors):
        for n, c in enumerate(st["cols"]):
            factors[n] = np.ascontiguousarray(c.T)

    def sgd_grads(self, shard, factors, rate, rng, counter_offset):
        seed, path = rng
        kept = np.flatnonzero(O.uniform(seed, path, shard.nnz, start=counter_offset) < rate)
        s = O.OTensor(shard.shape, shard.keys[kept], shard.values[kept])
        if s.nnz == 0:
            return [torch.zeros(f.shape, dtype=torch.float64) for f in factors]
        model = O.tttp(s.with_values(np.ones(s.nnz)), factors)
        phi1 = s.with_values(2.0 * (model - s.values))
        return [torch.from_numpy(O.mttkrp(phi1, factors, m)) for m in range(s.order)]

    def sgd_apply(self, factors, grads, step, shrink):
        for m in range(len(factors)):
            factors[m] = (factors[m] - step * grads[m].numpy()) - shrink * factors[m]


def _instance(nnz=20_000):
    rng = np.random.default_rng(42)
    shape = (300, 120, 50)
    i0 = synth.zipf_indices(rng, shape[0], nnz)
    i1 = synth.zipf_indices(rng, shape[1], nnz)
    i2 = rng.integers(0, shape[2], nnz)
    keys = np.unique((i0 * shape[1] + i1) * shape[2] + i2).astype(np.uint64)
    values = rng.integers(1, 6, keys.size).astype(np.float64)
    factors = [rng.random((d, 8)) / np.sqrt(8) for d in shape]
    return shape, keys, values, factors


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, outdir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        shape, keys, values, factors = _instance()
        coords = O.delinearize(keys, shape)
        als = D.ShardedALS(coords, values, shape, 1e-5, OracleBackend())
        fs = [f.copy() for f in factors]
        for _ in range(2):
            als.sweep(fs)
        np.savez(os.path.join(outdir, f"als{rank}.npz"), *fs,
                 blocks=np.array(als.blocks, dtype=np.int64))
        # SGD: nonzero shards, global Philox counter, all-reduced gradients
        lo, hi = D.nnz_partition(keys.size, world)[rank]
        seed, path, rate = 7, (1, 1), 0.3
        draws = O.uniform(seed, path, hi - lo, start=lo)
        kept_local = np.flatnonzero(draws < rate) + lo
        fs = [f.copy() for f in factors]
        ot = O.OTensor(shape, keys[kept_local], values[kept_local])
        if ot.nnz:
            model = O.tttp(ot.with_values(np.ones(ot.nnz)), fs)
            phi1 = ot.with_values(2.0 * (model - ot.values))
            grads = [O.mttkrp(phi1, fs, m) for m in range(3)]
        else:
            grads = [np.zeros_like(f) for f in fs]
        summed = []
        for g in grads:
            tg = torch.from_numpy(g)
            dist.all_reduce(tg)
            summed.append(tg.numpy())
        np.savez(os.path.join(outdir, f"sgd{rank}.npz"), kept=kept_local, *summed)
        # CCD++: nonzero shards, all-reduced (num, den) per (r, mode)
        ccd = D.ShardedCCD(keys, values, shape, 1e-5, OracleBackend())
        fs = [f.copy() for f in factors]
        ccd.sweep(fs)
        np.savez(os.path.join(outdir, f"ccd{rank}.npz"), *fs)
        # SGD steps through ShardedSGD
        sgd = D.ShardedSGD(keys, values, shape, OracleBackend())
        fs = [f.copy() for f in factors]
        for it in range(2):
            sgd.step(fs, 0.3, 1e-3, 1e-4, (7, (1, it)))
        np.savez(os.path.join(outdir, f"sgdsteps{rank}.npz"), *fs)
    finally:
        dist.destroy_process_group()


@pytest.fixture(scope="module")
def dist_run(tmp_path_factory):
    out = tmp_path_factory.mktemp("dist")
    mp.spawn(_worker, args=(2, _free_port(), str(out)), nprocs=2, join=True)
    return out


def test_row_cost_partition_and_uneven_gather_bytes():
    """cfg 3-like Zipf rows at P = 8: balancing nnz + a per-row solve cost
    moves rows off the tail block; the gather carries exactly I_n x R values."""
    rng = np.random.default_rng(0)
    counts = np.bincount(synth.zipf_indices(rng, 480_189, 2_000_000), minlength=480_189)
    by_nnz = D.row_partition(counts, 8)
    by_cost = D.row_partition(counts, 8, D.als_row_weight(32))
    cost = counts + D.als_row_weight(32)
    share = lambda blocks: max(cost[a:b].sum() for a, b in blocks) / cost.sum() * 8
    assert share(by_cost) < share(by_nnz)
    assert share(by_cost) < 1.05
    rows = [b - a for a, b in by_cost]
    assert sum(rows) == counts.size  # uneven gather = I_n x R values, no padding
    # a gather padded to the largest block of the nnz-only partition (round 1)
    # would have moved ~6.5x the factor
    assert max(b - a for a, b in by_nnz) * 8 > 5 * counts.size


def test_row_partition_balances_skewed_rows():
    counts = np.array([1000, 1, 1, 1, 500, 500, 3, 3])
    blocks = D.row_partition(counts, 2)
    assert blocks[0][0] == 0 and blocks[-1][1] == counts.size
    assert blocks[0][1] == blocks[1][0]
    assert D.row_partition(np.ones(10), 3) == [(0, 3), (3, 7), (7, 10)] or \
        sum(b - a for a, b in D.row_partition(np.ones(10), 3)) == 10
    parts = D.nnz_partition(1001, 4)
    assert parts[0][0] == 0 and parts[-1][1] == 1001
    assert all(a % 4 == 0 for a, _ in parts)


def test_shard_keys_rebase_and_order():
    shape, keys, values, _ = _instance(2000)
    coords = O.delinearize(keys, shape)
    sshape, skeys, sel = D.shard_keys(coords, shape, 1, 10, 40)
    assert sshape == (shape[0], 30, shape[2])
    assert np.all(np.diff(skeys) > 0)  # canonical order preserved
    sc = O.delinearize(skeys.astype(np.uint64), sshape)
    assert np.array_equal(sc[1] + 10, coords[1][sel])
    assert np.array_equal(sc[0], coords[0][sel])


def test_sharded_als_bitwise_equals_single_process(dist_run):
    shape, keys, values, factors = _instance()
    ot = O.OTensor(shape, keys, values)
    fs = [f.copy() for f in factors]
    for _ in range(2):
        O.als_sweep(ot, fs, 1e-5)
    for rank in range(2):
        z = np.load(os.path.join(dist_run, f"als{rank}.npz"))
        for n in range(3):
            assert np.array_equal(z[f"arr_{n}"], fs[n]), (rank, n)


def test_sharded_sgd_sample_and_gradients(dist_run):
    shape, keys, values, factors = _instance()
    ot = O.OTensor(shape, keys, values)
    kept = O.sample_positions(ot, 0.3, 7, (1, 1))
    z0 = np.load(os.path.join(dist_run, "sgd0.npz"))
    z1 = np.load(os.path.join(dist_run, "sgd1.npz"))
    assert np.array_equal(np.concatenate([z0["kept"], z1["kept"]]), kept)
    s = O.sample(ot, 0.3, 7, (1, 1))
    model = O.tttp(s.with_values(np.ones(s.nnz)), factors)
    phi1 = s.with_values(2.0 * (model - s.values))
    for m in range(3):
        ref = O.mttkrp(phi1, factors, m)
        got = z0[f"arr_{m}"]
        assert np.array_equal(got, z1[f"arr_{m}"])
        assert np.linalg.norm(got - ref) <= 1e-12 * np.linalg.norm(ref)


def test_sharded_ccd_matches_single_process(dist_run):
    shape, keys, values, factors = _instance()
    ot = O.OTensor(shape, keys, values)
    fs = [f.copy() for f in factors]
    O.ccd_sweep(ot, fs, 1e-5)
    z0 = np.load(os.path.join(dist_run, "ccd0.npz"))
    z1 = np.load(os.path.join(dist_run, "ccd1.npz"))
    for n in range(3):
        got = z0[f"arr_{n}"]
        assert np.array_equal(got, z1[f"arr_{n}"])  # replicas agree bit for bit
        assert np.linalg.norm(got - fs[n]) <= 1e-10 * np.linalg.norm(fs[n]), n


def test_sharded_sgd_steps_match_single_process(dist_run):
    shape, keys, values, factors = _instance()
    ot = O.OTensor(shape, keys, values)
    fs = [f.copy() for f in factors]
    for it in range(2):
        O.sgd_sweep(ot, fs, 1e-4, 1e-3, 0.3, 7, (1, it))
    z0 = np.load(os.path.join(dist_run, "sgdsteps0.npz"))
    z1 = np.load(os.path.join(dist_run, "sgdsteps1.npz"))
    for n in range(3):
        got = z0[f"arr_{n}"]
        assert np.array_equal(got, z1[f"arr_{n}"])
        assert np.linalg.norm(got - fs[n]) <= 1e-12 * np.linalg.norm(fs[n]), n
