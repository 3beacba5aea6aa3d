"""cProfile of the public numpy API calls (host-side overhead per call)."""
import cProfile
import os
import pstats
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1910_02371_b200 as cp  # noqa: E402
from paper_1910_02371_b200 import synth  # noqa: E402

shape, keys, values, factors = synth.cfg2()
pf = [torch.from_numpy(f).pin_memory() for f in factors]
hf = [p.numpy() for p in pf]
t = cp.SparseTensor(shape, keys, values)
for _ in range(3):
    cp.tttp(t, hf).values
    [cp.mttkrp(t, hf, m) for m in range(3)]
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
for _ in range(20):
    cp.tttp(t, hf).values
    [cp.mttkrp(t, hf, m) for m in range(3)]
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(25)
