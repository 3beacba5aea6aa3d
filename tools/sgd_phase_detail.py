"""Wall vs device time of the pieces of one SGD step at cfg 5 scale."""
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1910_02371_b200 as cp  # noqa: E402
from paper_1910_02371_b200 import synth  # noqa: E402
from paper_1910_02371_b200.core import _Shared, SparseTensor  # noqa: E402
from paper_1910_02371_b200.losses import tttp_affine  # noqa: E402
from paper_1910_02371_b200.optim import SolverConfig, _sgd_ls_device  # noqa: E402
from paper_1910_02371_b200.sampling import gather_values, sample_pattern  # noqa: E402

nnz = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000_000
shape, tn, values, F = synth.cfg5_device(nnz=nnz)
t = tn.with_values(values)
cfg = SolverConfig(rank=64, algorithm="sgd", step=1e-3, reg=1e-4, sample_rate=0.01)
for it in range(2):
    _sgd_ls_device(t, F, cfg, cp.RngState(5).child(1).child(it))
torch.cuda.synchronize()
res = {}


def timed(name, fn):
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    w0 = time.perf_counter()
    a.record()
    r = fn()
    w1 = time.perf_counter()
    b.record()
    torch.cuda.synchronize()
    w2 = time.perf_counter()
    res[name] = {"launch_wall_ms": round((w1 - w0) * 1e3, 3),
                 "total_wall_ms": round((w2 - w0) * 1e3, 3),
                 "device_ms": round(a.elapsed_time(b), 3)}
    return r


rng = cp.RngState(5).child(1).child(7)
pat, parent = timed("sample_pattern", lambda: sample_pattern(t, 0.01, rng))
vals = timed("gather_values", lambda: gather_values(t.device_values(torch.float32), parent))
sampled = SparseTensor._device_born(shape, pat.nnz, _Shared(pattern=pat), vals)
timed("tttp_affine", lambda: tttp_affine(sampled, F, 2.0, -2.0, torch.float32))
timed("tttp_affine_again", lambda: tttp_affine(sampled, F, 2.0, -2.0, torch.float32))
timed("full_step", lambda: _sgd_ls_device(t, F, cfg, cp.RngState(5).child(1).child(8)))
timed("full_step2", lambda: _sgd_ls_device(t, F, cfg, cp.RngState(5).child(1).child(9)))
print(json.dumps(res, indent=1))
