"""A few cfg 5 SGD steps for an ncu launch list (per-kernel times of one step)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1910_02371_b200 as cp  # noqa: E402
from paper_1910_02371_b200 import synth  # noqa: E402
from paper_1910_02371_b200.optim import SolverConfig, _sgd_ls_device  # noqa: E402

nnz = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000_000
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
shape, tn, values, F = synth.cfg5_device(nnz=nnz)
t = tn.with_values(values)
cfg = SolverConfig(rank=64, algorithm="sgd", step=1e-3, reg=1e-4, sample_rate=0.01)
for it in range(steps):
    _sgd_ls_device(t, F, cfg, cp.RngState(5).child(1).child(it))
torch.cuda.synchronize()
print("ok")
