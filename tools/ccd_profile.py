"""One CCD++ sweep at cfg 3 shape (nnz from argv), for ncu launch lists."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1910_02371_b200 as cp  # noqa: E402
from paper_1910_02371_b200 import synth  # noqa: E402
from paper_1910_02371_b200.optim import _ccd_ls_device  # noqa: E402

nnz = int(sys.argv[1]) if len(sys.argv) > 1 else 10_000_000
rank = int(sys.argv[2]) if len(sys.argv) > 2 else 4
shape, keys, vals = synth.cfg3_device(nnz=nnz)
t = cp.SparseTensor.from_device(shape, keys, vals)
g = np.random.default_rng(0)
F = [torch.from_numpy(g.random((d, rank)) / np.sqrt(rank)).cuda() for d in shape]
_ccd_ls_device(t, F, 1e-5)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
_ccd_ls_device(t, F, 1e-5)
e1.record()
torch.cuda.synchronize()
print("ccd sweep ms", e0.elapsed_time(e1), "passes", 3 * rank)
