"""MTTKRP time vs task size (entries per segmented task) at cfg 2 and a
cfg 3-like shape (CUDA events)."""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1910_02371_b200 as cp  # noqa: E402
from paper_1910_02371_b200 import _lib, synth  # noqa: E402

shape, keys, values, factors = synth.cfg2()
for ts in (256, 384, 512, 768, 1024, 2048):
    t = cp.SparseTensor(shape, keys, values, validate=False)
    t.set_task_size(ts)
    F = [torch.from_numpy(f).cuda() for f in factors]
    L = _lib.load()
    pat = t.device_pattern()
    s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    sv = [t.sorted_values(m, torch.float64) for m in range(3)]
    fp = _lib.ptr_array([f.data_ptr() for f in F])
    mo = [torch.empty(d, 16, dtype=torch.float64, device="cuda") for d in shape]
    res = []
    for m in range(3):
        def call():
            _lib.check(L.cpfit_mttkrp(pat.handle, m, 0, 16, ctypes.c_void_p(sv[m].data_ptr()), 1,
                                      fp, ctypes.c_void_p(mo[m].data_ptr()), s))
        for _ in range(3):
            call()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(20):
            call()
        b.record()
        torch.cuda.synchronize()
        res.append(round(a.elapsed_time(b) / 20, 4))
    print("task_size", ts, "mttkrp ms", res, flush=True)
