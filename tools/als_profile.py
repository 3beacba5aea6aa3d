"""Per-phase timing of one ALS sweep at BASELINE cfg 3 scale (CUDA events):
MTTKRP, Gram assembly and batched solve per mode, plus layout statistics."""
import ctypes
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1910_02371_b200 as cp  # noqa: E402
from paper_1910_02371_b200 import _lib, synth  # noqa: E402
from paper_1910_02371_b200.kernels import _ptrs  # noqa: E402
from paper_1910_02371_b200.optim import _als_ls_device  # noqa: E402

nnz = int(sys.argv[1]) if len(sys.argv) > 1 else 100_480_507
R, REG = 32, 1e-5
shape, keys, vals = synth.cfg3_device(nnz=nnz)
t = cp.SparseTensor.from_device(shape, keys, vals)
g = cp.RngState(0).child(0).generator()
F = [torch.from_numpy(g.random((d, R)) / np.sqrt(R)).cuda() for d in shape]
_als_ls_device(t, F, REG)
torch.cuda.synchronize()
L = _lib.load()
pat = t.device_pattern()
s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def ev():
    e = torch.cuda.Event(enable_timing=True)
    e.record()
    return e


res = {}
for mode in range(3):
    nt, ns, nsl = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
    L.cpfit_pattern_mode_stats(pat.handle, mode, s, ctypes.byref(nt), ctypes.byref(ns),
                               ctypes.byref(nsl))
    ptrs = _ptrs([None if n == mode else f for n, f in enumerate(F)])
    rhs = torch.empty(shape[mode], R, dtype=torch.float64, device="cuda")
    gram = torch.empty(shape[mode], R, R, dtype=torch.float64, device="cuda")
    x = torch.empty_like(rhs)
    sv = t.sorted_values(mode)
    out = {"ntasks": nt.value, "nsplit": ns.value, "nslots": nsl.value}
    for rep in range(2):
        e0 = ev()
        _lib.check(L.cpfit_mttkrp(pat.handle, mode, 0, R, ctypes.c_void_p(sv.data_ptr()), 1, ptrs,
                                  ctypes.c_void_p(rhs.data_ptr()), s))
        e1 = ev()
        _lib.check(L.cpfit_gram(pat.handle, mode, 0, R, None, 1, ptrs,
                                ctypes.c_void_p(gram.data_ptr()), s))
        e2 = ev()
        bad = ctypes.c_int64()
        _lib.check(L.cpfit_solve_factor(pat.handle, mode, 0, R, None, 1, ptrs,
                                        ctypes.c_void_p(rhs.data_ptr()), REG,
                                        ctypes.c_void_p(x.data_ptr()), None,
                                        ctypes.byref(bad), s))
        e3 = ev()
        torch.cuda.synchronize()
    out["mttkrp_ms"] = e0.elapsed_time(e1)
    out["gram_ms"] = e1.elapsed_time(e2)
    out["gram_plus_solve_ms"] = e2.elapsed_time(e3)
    out["solve_only_ms_est"] = out["gram_plus_solve_ms"] - out["gram_ms"]
    flop = t.nnz * (R + R * (R + 1))  # SURVEY 8d Gram flops (N=3)
    out["gram_gflops"] = flop / (out["gram_ms"] * 1e-3) / 1e9
    res[f"mode{mode}"] = out
print(json.dumps(res, indent=1))
