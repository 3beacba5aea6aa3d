"""Does numpy-API traffic before SGD steps slow them down?  Variant from argv:
none | tttp | mttkrp | both."""
import gc
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1910_02371_b200 as cp  # noqa: E402
from paper_1910_02371_b200 import synth  # noqa: E402
from paper_1910_02371_b200.optim import SolverConfig, _sgd_ls_device  # noqa: E402

variant = sys.argv[1] if len(sys.argv) > 1 else "none"
if variant != "none":
    shape, keys, values, factors = synth.cfg2()
    pv = torch.from_numpy(values).pin_memory()
    pf = [torch.from_numpy(f).pin_memory() for f in factors]
    t2 = cp.SparseTensor(shape, keys, pv.numpy(), validate=False)
    hf = [p.numpy() for p in pf]
    for _ in range(10):
        if variant in ("tttp", "both"):
            o = cp.tttp(t2, hf)
        if variant in ("mttkrp", "both"):
            [cp.mttkrp(t2, hf, m) for m in range(3)]
        if variant in ("tttp", "both"):
            o.values
    del t2
    o = None
    gc.collect()
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
shape, tn, values, F = synth.cfg5_device()
t = tn.with_values(values)
cfg = SolverConfig(rank=64, algorithm="sgd", step=1e-3, reg=1e-4, sample_rate=0.01)
root = cp.RngState(5).child(1)
for it in range(2):
    _sgd_ls_device(t, F, cfg, root.child(100 + it))
torch.cuda.synchronize()
ms = []
for it in range(6):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    _sgd_ls_device(t, F, cfg, root.child(it))
    b.record()
    torch.cuda.synchronize()
    ms.append(round(a.elapsed_time(b), 1))
print(variant, ms, flush=True)
