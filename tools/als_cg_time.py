"""cfg 3 implicit-CG ALS sweep next to the direct (Gram + Cholesky) sweep:
per-mode time, CG iterations, peak memory, rmse after each."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1910_02371_b200 as cp  # noqa: E402
from paper_1910_02371_b200 import synth  # noqa: E402
from paper_1910_02371_b200.optim import _als_ls_device, _als_mode_cg_device  # noqa: E402

nnz = int(sys.argv[1]) if len(sys.argv) > 1 else 100_480_507
tol = float(sys.argv[2]) if len(sys.argv) > 2 else 5e-3
R = 32
shape, keys, vals = synth.cfg3_device(nnz=nnz)
t = cp.SparseTensor.from_device(shape, keys, vals)
g = cp.RngState(0).child(0).generator()
F0 = [torch.from_numpy(g.random((d, R)) / np.sqrt(R)).cuda() for d in shape]


def timed(fn):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    r = fn()
    e1.record()
    torch.cuda.synchronize()
    return r, e0.elapsed_time(e1)


out = {"nnz": nnz, "rank": R, "cg_tol": tol, "cg_max": min(30, 3 * R)}
for solver in ("direct", "cg"):
    F = [f.clone() for f in F0]
    torch.cuda.reset_peak_memory_stats()
    base = torch.cuda.memory_allocated()
    sweeps = []
    for sweep in range(4):
        modes = []
        for mode in range(3):
            if solver == "direct":
                from paper_1910_02371_b200.optim import _als_mode_device
                x, ms = timed(lambda: _als_mode_device(t, F, mode, 1e-5))
                modes.append({"ms": ms})
            else:
                (x, _, it), ms = timed(lambda: _als_mode_cg_device(t, F, mode, 1e-5, tol,
                                                                   min(30, 3 * R)))
                modes.append({"ms": ms, "iters": it})
            F[mode] = x
        sweeps.append({"modes": modes, "sweep_ms": sum(m["ms"] for m in modes),
                       "rmse": float(cp.rmse(t, F))})
    out[solver] = {"sweeps": sweeps,
                   "peak_extra_GB": (torch.cuda.max_memory_allocated() - base) / 1e9}
print(json.dumps(out, indent=1))
