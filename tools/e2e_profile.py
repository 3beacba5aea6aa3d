"""Break the bench e2e step (cfg 2 via the public numpy API) into its parts:
each API call's wall time and the raw PCIe copy rates it is bounded by."""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1910_02371_b200 as cp  # noqa: E402
from paper_1910_02371_b200 import synth  # noqa: E402

shape, keys, values, factors = synth.cfg2()
pv = torch.from_numpy(values).pin_memory()
pf = [torch.from_numpy(f).pin_memory() for f in factors]
hv, hf = pv.numpy(), [p.numpy() for p in pf]
t = cp.SparseTensor(shape, keys, hv)
for _ in range(2):
    cp.tttp(t, hf).values
    [cp.mttkrp(t, hf, m) for m in range(3)]
torch.cuda.synchronize()


def wall(fn, n=5):
    ts = []
    for _ in range(n):
        torch.cuda.synchronize()
        a = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        ts.append((time.perf_counter() - a) * 1e3)
    return float(np.median(ts))


res = {}
res["tttp_api_incl_values_ms"] = wall(lambda: cp.tttp(t, hf).values)
res["tttp_api_device_only_ms"] = wall(lambda: cp.tttp(t, [torch.from_numpy(f).cuda() for f in hf]))
for m in range(3):
    res[f"mttkrp{m}_api_ms"] = wall(lambda: cp.mttkrp(t, hf, m))
dv = torch.empty(t.nnz, dtype=torch.float64, device="cuda")
hp = torch.empty(t.nnz, dtype=torch.float64, pin_memory=True)
res["d2h_80MB_pinned_ms"] = wall(lambda: hp.copy_(dv))
hpage = np.empty(t.nnz)
res["d2h_80MB_pageable_ms"] = wall(lambda: hpage.__setitem__(slice(None), dv.cpu().numpy()))
df = torch.empty(factors[0].shape, dtype=torch.float64, device="cuda")
res["h2d_factor_pinned_ms"] = wall(lambda: df.copy_(pf[0]))
res["h2d_factor_from_numpy_ms"] = wall(lambda: torch.from_numpy(hf[0]).to("cuda"))
res["alloc_pinned_80MB_ms"] = wall(lambda: torch.empty(t.nnz, dtype=torch.float64, pin_memory=True))
res["step_ms"] = wall(lambda: (cp.tttp(t, hf).values, [cp.mttkrp(t, hf, m) for m in range(3)]))
print(json.dumps(res, indent=1))


def step_parts(n=5):
    """Wall time to each point of one bench e2e step (ms)."""
    rows = []
    for _ in range(n):
        torch.cuda.synchronize()
        a = time.perf_counter()
        out = cp.tttp(t, hf)
        b = time.perf_counter()
        ms_ = [cp.mttkrp(t, hf, m) for m in range(3)]
        c = time.perf_counter()
        v = out.values
        d = time.perf_counter()
        torch.cuda.synchronize()
        rows.append(((b - a) * 1e3, (c - b) * 1e3, (d - c) * 1e3, (d - a) * 1e3))
    return [float(x) for x in np.median(np.array(rows), axis=0)]


res["step_tttp_return_mttkrps_values_total_ms"] = step_parts()
print(json.dumps(res, indent=1))


def step_parts2(n=5):
    rows = []
    for _ in range(n):
        torch.cuda.synchronize()
        ts = [time.perf_counter()]
        out = cp.tttp(t, hf)
        ts.append(time.perf_counter())
        for m in range(3):
            cp.mttkrp(t, hf, m)
            ts.append(time.perf_counter())
        out.values
        ts.append(time.perf_counter())
        rows.append(np.diff(ts) * 1e3)
    return [float(x) for x in np.median(np.array(rows), axis=0)]


def mttkrp_inside(n=5):
    """One mttkrp call while an 80 MB D2H drains on another stream."""
    cs = torch.cuda.Stream()
    dv = torch.empty(t.nnz, dtype=torch.float64, device="cuda")
    hp = torch.empty(t.nnz, dtype=torch.float64, pin_memory=True)
    rows = []
    for _ in range(n):
        torch.cuda.synchronize()
        with torch.cuda.stream(cs):
            hp.copy_(dv, non_blocking=True)
        a = time.perf_counter()
        cp.mttkrp(t, hf, 0)
        b = time.perf_counter()
        torch.cuda.synchronize()
        rows.append((b - a) * 1e3)
    return float(np.median(rows))


res2 = {"per_call_ms": step_parts2(), "mttkrp_during_d2h_ms": mttkrp_inside()}
print(json.dumps(res2, indent=1))
