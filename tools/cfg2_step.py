"""A few cfg 2 steps (TTTP + MTTKRP x3, fp64, R=16) for ncu captures."""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1910_02371_b200 as cp  # noqa: E402
from paper_1910_02371_b200 import _lib, synth  # noqa: E402

shape, keys, values, factors = synth.cfg2()
t = cp.SparseTensor(shape, keys, values, validate=False)
F = [torch.from_numpy(f).cuda() for f in factors]
L = _lib.load()
pat = t.device_pattern()
s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
vals = t.device_values(torch.float64)
sv = [t.sorted_values(m, torch.float64) for m in range(3)]
fp = _lib.ptr_array([f.data_ptr() for f in F])
out = torch.empty(t.nnz, dtype=torch.float64, device="cuda")
mo = [torch.empty(d, 16, dtype=torch.float64, device="cuda") for d in shape]
for _ in range(int(sys.argv[1]) if len(sys.argv) > 1 else 3):
    _lib.check(L.cpfit_tttp(pat.handle, 0, 16, ctypes.c_void_p(vals.data_ptr()), fp,
                            ctypes.c_void_p(out.data_ptr()), s))
    for m in range(3):
        _lib.check(L.cpfit_mttkrp(pat.handle, m, 0, 16, ctypes.c_void_p(sv[m].data_ptr()), 1, fp,
                                  ctypes.c_void_p(mo[m].data_ptr()), s))
torch.cuda.synchronize()
print("ok")
