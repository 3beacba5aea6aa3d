"""Host-side cost of the numpy API calls (cProfile over repeated calls)."""
import cProfile
import os
import pstats
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1910_02371_b200 as cp  # noqa: E402
from paper_1910_02371_b200 import synth  # noqa: E402

shape, keys, values, factors = synth.cfg2()
pv = torch.from_numpy(values).pin_memory()
pf = [torch.from_numpy(f).pin_memory() for f in factors]
t = cp.SparseTensor(shape, keys, pv.numpy(), validate=False)
hf = [p.numpy() for p in pf]


def step():
    o = cp.tttp(t, hf)
    [cp.mttkrp(t, hf, m) for m in range(3)]
    o.values


for _ in range(3):
    step()
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
for _ in range(20):
    step()
torch.cuda.synchronize()
pr.disable()
st = pstats.Stats(pr)
st.sort_stats("tottime").print_stats(18)
