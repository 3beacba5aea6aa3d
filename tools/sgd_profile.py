"""Phase timing of one SGD step at BASELINE cfg 5 scale (1e9 nnz by default):
sample, value gather, derivative TTTP, per-mode layout build + MTTKRP, update."""
import ctypes
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1910_02371_b200 as cp  # noqa: E402
from paper_1910_02371_b200 import _lib, synth  # noqa: E402
from paper_1910_02371_b200.core import _Shared, SparseTensor  # noqa: E402
from paper_1910_02371_b200.kernels import _ptrs  # noqa: E402
from paper_1910_02371_b200.losses import tttp_affine  # noqa: E402
from paper_1910_02371_b200.sampling import gather_values, sample_pattern  # noqa: E402

nnz = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000_000
shape, tn, values, F = synth.cfg5_device(nnz=nnz)
t = tn.with_values(values)
L = _lib.load()
s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
res = {}
for it in range(3):
    rng = cp.RngState(5).child(1).child(it)
    torch.cuda.synchronize()
    ev = []

    def mark(name):
        torch.cuda.synchronize()
        ev.append((name, time.perf_counter()))
    mark("start")
    pat, parent = sample_pattern(t, 0.01, rng)
    mark("sample")
    vals = gather_values(t.device_values(torch.float32), parent)
    mark("gather_values")
    sampled = SparseTensor._device_born(shape, pat.nnz, _Shared(pattern=pat), vals)
    phi1 = tttp_affine(sampled, F, 2.0, -2.0, torch.float32)
    mark("tttp_deriv")
    for mode in range(4):
        nt = ctypes.c_int64()
        L.cpfit_pattern_mode_stats(pat.handle, mode, s, ctypes.byref(nt), None, None)
        mark(f"layout{mode}")
        g = torch.empty((shape[mode], 64), dtype=torch.float32, device="cuda")
        _lib.check(L.cpfit_mttkrp(pat.handle, mode, 1, 64, ctypes.c_void_p(phi1.data_ptr()), 0,
                                  _ptrs(F), ctypes.c_void_p(g.data_ptr()), s))
        mark(f"mttkrp{mode}")
    res = {b[0]: round((b[1] - a[1]) * 1e3, 3) for a, b in zip(ev[:-1], ev[1:])}
    res["sample_nnz"] = pat.nnz
print(json.dumps(res))
