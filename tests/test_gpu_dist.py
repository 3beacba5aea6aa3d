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
