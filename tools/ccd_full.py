"""cfg 3 CCD++ sweep at R=32 (the bench's number), twice."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1910_02371_b200 as cp  # noqa: E402
from paper_1910_02371_b200 import synth  # noqa: E402
from paper_1910_02371_b200.optim import _ccd_ls_device  # noqa: E402

shape, keys, vals = synth.cfg3_device()
t = cp.SparseTensor.from_device(shape, keys, vals)
g = cp.RngState(0).child(0).generator()
F0 = [torch.from_numpy(g.random((d, 32)) / np.sqrt(32)).cuda() for d in shape]
for rep in range(3):
    F = [f.clone() for f in F0]
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    _ccd_ls_device(t, F, 1e-5)
    e1.record()
    torch.cuda.synchronize()
    print("ccd sweep ms", e0.elapsed_time(e1), "checksum", float(sum(f.sum() for f in F)))
