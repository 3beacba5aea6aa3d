"""cfg 3 direct ALS: per-mode update times (CUDA events) of sweeps 2-4."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1910_02371_b200 as cp  # noqa: E402
from paper_1910_02371_b200 import synth  # noqa: E402
from paper_1910_02371_b200.optim import _als_mode_device  # noqa: E402

nnz = int(sys.argv[1]) if len(sys.argv) > 1 else 100_480_507
keep = len(sys.argv) > 2 and sys.argv[2] == "keep"
R = 32
shape, keys, vals = synth.cfg3_device(nnz=nnz)
t = cp.SparseTensor.from_device(shape, keys, vals)
g = cp.RngState(0).child(0).generator()
F = [torch.from_numpy(g.random((d, R)) / np.sqrt(R)).cuda() for d in shape]
res = []
for sweep in range(4):
    ms = []
    for mode in range(3):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        out = _als_mode_device(t, F, mode, 1e-5, keep_gram=keep)
        e1.record()
        torch.cuda.synchronize()
        F[mode] = out[0] if keep else out
        ms.append(round(e0.elapsed_time(e1), 3))
    res.append(ms)
print(json.dumps({"env_line": os.environ.get("CPFIT_GRAM_LINE"), "modes_ms": res[1:],
                  "sweep_ms": [round(sum(m), 3) for m in res[1:]]}))
