"""What slows the MTTKRP API calls while the 80 MB TTTP-values D2H drains?
Times, with and without a concurrent 80 MB device->host DMA on another stream:
a 1.28 MB H2D factor upload, a 1.28 MB SM-driven pinned write, and the MTTKRP
API with device / numpy factors (cfg 2)."""
import ctypes
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1910_02371_b200 as cp  # noqa: E402
from paper_1910_02371_b200 import _lib, synth  # noqa: E402
from paper_1910_02371_b200.core import to_host_sm  # noqa: E402

shape, keys, values, factors = synth.cfg2()
t = cp.SparseTensor(shape, keys, values, validate=False)
pf = [torch.from_numpy(f).pin_memory() for f in factors]
hf = [p.numpy() for p in pf]
df = [p.cuda() for p in pf]
for m in range(3):
    cp.mttkrp(t, hf, m)
cs = torch.cuda.Stream()
dv = torch.empty(t.nnz, dtype=torch.float64, device="cuda")
hp = torch.empty(t.nnz, dtype=torch.float64, pin_memory=True)
dres = torch.randn(10000, 16, dtype=torch.float64, device="cuda")
dst = torch.empty_like(df[0])


def run(fn, busy, n=7):
    rows = []
    for _ in range(n):
        torch.cuda.synchronize()
        if busy:
            with torch.cuda.stream(cs):
                hp.copy_(dv, non_blocking=True)
        a = time.perf_counter()
        fn()
        rows.append((time.perf_counter() - a) * 1e3)
        torch.cuda.synchronize()
    return round(float(np.median(rows)), 3)


def h2d():
    dst.copy_(pf[0], non_blocking=True)
    torch.cuda.current_stream().synchronize()


cases = {
    "h2d_1.28MB_sync": h2d,
    "sm_pinned_write_1.28MB": lambda: to_host_sm(dres),
    "mttkrp_api_device_factors_numpy_out": lambda: to_host_sm(cp.mttkrp(t, df, 0)),
    "mttkrp_api_numpy_factors": lambda: cp.mttkrp(t, hf, 0),
    "kernel_only_sync": lambda: (cp.mttkrp(t, df, 0), torch.cuda.current_stream().synchronize()),
}
out = {k: {"idle_ms": run(f, False), "during_d2h_ms": run(f, True)} for k, f in cases.items()}
print(json.dumps(out, indent=1))
