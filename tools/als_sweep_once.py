"""Two ALS sweeps at cfg 3 (the second is the one to read in a launch list)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1910_02371_b200 as cp  # noqa: E402
from paper_1910_02371_b200 import synth  # noqa: E402
from paper_1910_02371_b200.optim import _als_ls_device  # noqa: E402

nnz = int(sys.argv[1]) if len(sys.argv) > 1 else 100_480_507
R = 32
shape, keys, vals = synth.cfg3_device(nnz=nnz)
t = cp.SparseTensor.from_device(shape, keys, vals)
g = cp.RngState(0).child(0).generator()
F = [torch.from_numpy(g.random((d, R)) / np.sqrt(R)).cuda() for d in shape]
_als_ls_device(t, F, 1e-5, keep_gram=False)
torch.cuda.synchronize()
torch.cuda.nvtx.range_push("sweep")
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
_als_ls_device(t, F, 1e-5, keep_gram=False)
e1.record()
torch.cuda.synchronize()
print("als sweep ms", e0.elapsed_time(e1))
