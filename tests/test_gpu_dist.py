"""The device (NCCL) backend of the row-sharded ALS on one GPU: a single-rank
NCCL group exercises the shard construction on the device (torch index
arithmetic, rebased keys, device patterns), the per-block solve with row
offsets and the all-gather; the result must equal the unsharded device sweep
bit for bit.  Multi-rank behaviour of the same algebra is covered on the CPU
(tests/test_dist.py, gloo, 2 ranks)."""

import os
import socket

import numpy as np
import pytest

import paper_1910_02371_b200 as cp
from paper_1910_02371_b200 import synth

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def test_sharded_als_device_backend_single_rank():
    import torch
    import torch.distributed as dist

    from paper_1910_02371_b200 import dist as D
    from paper_1910_02371_b200.optim import _als_ls_device
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(_free_port())
    dist.init_process_group("nccl", rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    try:
        shape, keys, vals = synth.cfg3_device(nnz=200_000, shape=(3000, 500, 80))
        coords = []
        rem = keys.clone()
        for d in reversed(shape):
            coords.append(rem % d)
            rem = rem // d
        coords = coords[::-1]
        g = np.random.default_rng(0)
        init = [torch.from_numpy(g.random((d, 16)) / 4.0).cuda() for d in shape]
        als = D.ShardedALS(coords, vals, shape, 1e-5, D.DeviceBackend())
        F1 = [f.clone() for f in init]
        als.sweep(F1)
        t = cp.SparseTensor.from_device(shape, keys, vals)
        F2 = [f.clone() for f in init]
        _als_ls_device(t, F2, 1e-5, keep_gram=False)
        for a, b in zip(F1, F2):
            assert torch.equal(a, b)
        # implicit-CG solver through the same sharding: equals the unsharded
        # CG sweep bit for bit (same kernels, rebased rows)
        from paper_1910_02371_b200.optim import _als_ls_cg_device
        alsc = D.ShardedALS(coords, vals, shape, 1e-5,
                            D.DeviceBackend(als_solver="cg", cg_tol=1e-6, cg_max=48))
        F3 = [f.clone() for f in init]
        alsc.sweep(F3)
        F4 = [f.clone() for f in init]
        _als_ls_cg_device(t, F4, 1e-5, 1e-6, 48)
        for a, b in zip(F3, F4):
            assert torch.equal(a, b)
    finally:
        dist.destroy_process_group()


def _nccl_single_rank():
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(_free_port())
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    return dist


def test_sharded_ccd_and_sgd_device_backend_single_rank():
    """ShardedCCD (cpfit_ccd_numden + cpfit_ccd_apply) and ShardedSGD on one
    rank equal the fused single-device CCD++ sweep / SGD step bit for bit."""
    import torch

    from paper_1910_02371_b200 import dist as D
    from paper_1910_02371_b200.optim import SolverConfig, _ccd_ls_device, _sgd_ls_device
    dist = _nccl_single_rank()
    try:
        shape, keys, vals = synth.cfg3_device(nnz=100_000, shape=(2000, 400, 60))
        g = np.random.default_rng(1)
        init = [torch.from_numpy(g.random((d, 8)) / 4.0).cuda() for d in shape]
        t = cp.SparseTensor.from_device(shape, keys, vals)
        ccd = D.ShardedCCD(keys, vals, shape, 1e-5, D.DeviceBackend())
        F1 = [f.clone() for f in init]
        ccd.sweep(F1)
        F2 = [f.clone() for f in init]
        _ccd_ls_device(t, F2, 1e-5)
        for a, b in zip(F1, F2):
            assert torch.equal(a, b)
        sgd = D.ShardedSGD(keys, vals, shape, D.DeviceBackend())
        cfg = SolverConfig(algorithm="sgd", rank=8, step=1e-3, reg=1e-4, sample_rate=0.05)
        F1 = [f.clone() for f in init]
        F2 = [f.clone() for f in init]
        for it in range(2):
            rng = cp.RngState(3).child(1).child(it)
            sgd.step(F1, cfg.sample_rate, cfg.step, cfg.reg, rng)
            _sgd_ls_device(t, F2, cfg, cp.RngState(3).child(1).child(it))
        for a, b in zip(F1, F2):
            assert torch.equal(a, b)
    finally:
        dist.destroy_process_group()


def _world2_device_worker(rank, world, port, outdir):
    """One of two ranks on the same GPU; collectives through gloo (host-side
    copies: no kernel of one rank waits on the other's)."""
    import torch
    import torch.distributed as dist

    from paper_1910_02371_b200 import dist as D
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        shape, keys, vals = synth.cfg3_device(nnz=200_000, shape=(3000, 500, 80))
        coords = []
        rem = keys.clone()
        for d in reversed(shape):
            coords.append(rem % d)
            rem = rem // d
        coords = coords[::-1]
        g = np.random.default_rng(0)
        init = [torch.from_numpy(g.random((d, 16)) / 4.0).cuda() for d in shape]
        als = D.ShardedALS(coords, vals, shape, 1e-5, D.DeviceBackend(), rank_r=16)
        F = [f.clone() for f in init]
        for _ in range(2):
            als.sweep(F)
        np.savez(os.path.join(outdir, f"als{rank}.npz"), *[f.cpu().numpy() for f in F],
                 blocks=np.array(als.blocks, dtype=np.int64))
        ccd = D.ShardedCCD(keys, vals, shape, 1e-5, D.DeviceBackend())
        F = [f.clone() for f in init]
        ccd.sweep(F)
        np.savez(os.path.join(outdir, f"ccd{rank}.npz"), *[f.cpu().numpy() for f in F])
        sgd = D.ShardedSGD(keys, vals, shape, D.DeviceBackend())
        F = [f.clone() for f in init]
        for it in range(2):
            sgd.step(F, 0.05, 1e-3, 1e-4, cp.RngState(3).child(1).child(it))
        np.savez(os.path.join(outdir, f"sgd{rank}.npz"), *[f.cpu().numpy() for f in F])
    finally:
        dist.destroy_process_group()


def test_world2_device_backend_on_one_gpu(tmp_path):
    """ShardedALS / ShardedCCD / ShardedSGD with the device backend at world
    size 2: ALS equals the single-device sweeps bit for bit (row-local algebra,
    uneven block gather), CCD++ / SGD within 1e-10 / 1e-12 (all-reduced sums
    reassociate), replicas bit-identical."""
    import torch
    import torch.multiprocessing as mp

    from paper_1910_02371_b200.optim import SolverConfig, _als_ls_device, _ccd_ls_device, \
        _sgd_ls_device
    mp.spawn(_world2_device_worker, args=(2, _free_port(), str(tmp_path)), nprocs=2, join=True)
    shape, keys, vals = synth.cfg3_device(nnz=200_000, shape=(3000, 500, 80))
    g = np.random.default_rng(0)
    init = [torch.from_numpy(g.random((d, 16)) / 4.0).cuda() for d in shape]
    t = cp.SparseTensor.from_device(shape, keys, vals)
    F = [f.clone() for f in init]
    for _ in range(2):
        _als_ls_device(t, F, 1e-5, keep_gram=False)
    z = [np.load(os.path.join(tmp_path, f"als{r}.npz")) for r in range(2)]
    blocks = z[0]["blocks"]
    assert blocks.shape == (3, 2, 2) and all(b[0][1] == b[1][0] for b in blocks)
    for n in range(3):
        for r in range(2):
            assert np.array_equal(z[r][f"arr_{n}"], F[n].cpu().numpy()), (r, n)
    F = [f.clone() for f in init]
    _ccd_ls_device(t, F, 1e-5)
    z = [np.load(os.path.join(tmp_path, f"ccd{r}.npz")) for r in range(2)]
    for n in range(3):
        ref = F[n].cpu().numpy()
        assert np.array_equal(z[0][f"arr_{n}"], z[1][f"arr_{n}"])
        assert np.linalg.norm(z[0][f"arr_{n}"] - ref) <= 1e-10 * np.linalg.norm(ref)
    cfg = SolverConfig(algorithm="sgd", rank=16, step=1e-3, reg=1e-4, sample_rate=0.05)
    F = [f.clone() for f in init]
    for it in range(2):
        _sgd_ls_device(t, F, cfg, cp.RngState(3).child(1).child(it))
    z = [np.load(os.path.join(tmp_path, f"sgd{r}.npz")) for r in range(2)]
    for n in range(3):
        ref = F[n].cpu().numpy()
        assert np.array_equal(z[0][f"arr_{n}"], z[1][f"arr_{n}"])
        assert np.linalg.norm(z[0][f"arr_{n}"] - ref) <= 1e-12 * np.linalg.norm(ref)
