"""One Gauss-Newton step at cfg 3 shape (nnz from argv, default full):
wall / device time, for the ncu launch list of its kernels."""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1910_02371_b200 as cp  # noqa: E402
from paper_1910_02371_b200 import synth  # noqa: E402
from paper_1910_02371_b200.losses import get_loss  # noqa: E402
from paper_1910_02371_b200.optim import CompletionState, SolverConfig, _als_ls_device  # noqa: E402
from paper_1910_02371_b200.second_order import gn_step_device  # noqa: E402

nnz = int(sys.argv[1]) if len(sys.argv) > 1 else 100_480_507
R = 32
shape, keys, vals = synth.cfg3_device(nnz=nnz)
t = cp.SparseTensor.from_device(shape, keys, vals)
g = cp.RngState(0).child(0).generator()
init = [torch.from_numpy(g.random((d, R)) / np.sqrt(R)).cuda() for d in shape]
cfg = SolverConfig(rank=R, reg=1e-5, gn_damping=1.0)
res = []
for rep in range(2):
    F = [f.clone() for f in init]
    _als_ls_device(t, F, 1e-5)
    st = CompletionState(factors=F, rng=cp.RngState(0))
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    w = time.perf_counter()
    a.record()
    cg = gn_step_device(t, F, get_loss("ls"), cfg, st, "gauss_newton")
    b.record()
    torch.cuda.synchronize()
    res.append({"cg": cg, "device_ms": a.elapsed_time(b), "wall_ms": (time.perf_counter() - w) * 1e3})
print(json.dumps(res))
