"""Characterise the gather ceiling: TTTP / MTTKRP at 1e7 nnz, R=16 fp64, with
factor tables from L1-resident (256 rows) to HBM-resident (4e6 rows)."""
import ctypes
import json
import sys
import os

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1910_02371_b200 as cp  # noqa: E402
from paper_1910_02371_b200 import _lib, synth  # noqa: E402

R = 16
NNZ = 10_000_000
res = []
for I in (256, 2000, 10_000, 100_000, 1_000_000, 4_000_000):
    rng = np.random.default_rng(I)
    keys = synth.distinct_uniform_keys(rng, I ** 3, NNZ)
    t = cp.SparseTensor((I, I, I), keys, rng.standard_normal(NNZ), validate=False)
    fs = [torch.randn(I, R, dtype=torch.float64, device="cuda") for _ in range(3)]
    L = _lib.load()
    pat = t.device_pattern()
    s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    vals = t.device_values()
    sv = [t.sorted_values(m) for m in range(3)]
    fp = _lib.ptr_array([f.data_ptr() for f in fs])
    out = torch.empty(NNZ, dtype=torch.float64, device="cuda")
    mo = [torch.empty(I, R, dtype=torch.float64, device="cuda") for _ in range(3)]

    def timeit(fn, n=20):
        for _ in range(3):
            fn()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(n):
            fn()
        b.record()
        torch.cuda.synchronize()
        return a.elapsed_time(b) / n

    tt = timeit(lambda: L.cpfit_tttp(pat.handle, 0, R, ctypes.c_void_p(vals.data_ptr()), fp,
                                     ctypes.c_void_p(out.data_ptr()), s))
    mt = [timeit(lambda m=m: L.cpfit_mttkrp(pat.handle, m, 0, R, ctypes.c_void_p(sv[m].data_ptr()),
                                           1, fp, ctypes.c_void_p(mo[m].data_ptr()), s))
          for m in range(3)]
    r = {"rows": I, "table_MB": I * R * 8 / 1e6, "tttp_ms": tt, "mttkrp_ms": mt,
         "tttp_gather_TBs": NNZ * 3 * R * 8 / tt / 1e9,
         "mttkrp_gather_TBs": [NNZ * 2 * R * 8 / x / 1e9 for x in mt]}
    print(json.dumps(r), flush=True)
    del t, pat
