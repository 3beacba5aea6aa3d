"""One Poisson inner-Newton ALS sweep at cfg 3 (for ncu launch lists)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1910_02371_b200 as cp  # noqa: E402
from paper_1910_02371_b200 import synth  # noqa: E402
from paper_1910_02371_b200.losses import get_loss  # noqa: E402
from paper_1910_02371_b200.optim import SolverConfig, _als_generalized_device  # noqa: E402

nnz = int(sys.argv[1]) if len(sys.argv) > 1 else 100_480_507
R = 32
shape, keys, vals = synth.cfg3_device(nnz=nnz)
t = cp.SparseTensor.from_device(shape, keys, vals)
g = cp.RngState(0).child(0).generator()
init = [torch.from_numpy(g.random((d, R)) / np.sqrt(R)).cuda() for d in shape]
cfg = SolverConfig(rank=R, reg=1e-5, loss="poisson")
loss = get_loss("poisson")
for rep in range(2):
    F = [f.clone() for f in init]
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    _als_generalized_device(t, F, loss, cfg)
    b.record()
    torch.cuda.synchronize()
    print("poisson als sweep ms", a.elapsed_time(b))
