"""cfg 3 TTTP + MTTKRP (fp64, R=32, full 1.005e8 Zipf nnz) and the cfg 5 TTTP
residual (fp32, R=64, 1e9 order-4 nnz) once each, for ncu captures."""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1910_02371_b200 as cp  # noqa: E402
from paper_1910_02371_b200 import _lib, synth  # noqa: E402
from paper_1910_02371_b200.losses import tttp_affine  # noqa: E402

L = _lib.load()
s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
which = sys.argv[1] if len(sys.argv) > 1 else "35"
if "3" in which:
    shape, keys, vals = synth.cfg3_device()
    t = cp.SparseTensor.from_device(shape, keys, vals)
    del keys
    g = cp.RngState(0).child(0).generator()
    F = [torch.from_numpy(g.random((d, 32)) / np.sqrt(32)).cuda() for d in shape]
    fp = _lib.ptr_array([f.data_ptr() for f in F])
    pat = t.device_pattern()
    v = t.device_values(torch.float64)
    sv = [t.sorted_values(m, torch.float64) for m in range(3)]
    out = torch.empty(t.nnz, dtype=torch.float64, device="cuda")
    mo = [torch.empty(d, 32, dtype=torch.float64, device="cuda") for d in shape]
    _lib.check(L.cpfit_tttp(pat.handle, 0, 32, ctypes.c_void_p(v.data_ptr()), fp,
                            ctypes.c_void_p(out.data_ptr()), s))
    for m in range(3):
        _lib.check(L.cpfit_mttkrp(pat.handle, m, 0, 32, ctypes.c_void_p(sv[m].data_ptr()), 1, fp,
                                  ctypes.c_void_p(mo[m].data_ptr()), s))
    torch.cuda.synchronize()
    del t, out, mo, sv, v, pat
    torch.cuda.empty_cache()
if "5" in which:
    shape, t, values, F = synth.cfg5_device()
    tv = t.with_values(values)
    resid = tttp_affine(tv, F, -1.0, 1.0, torch.float32)
    torch.cuda.synchronize()
print("ok")
