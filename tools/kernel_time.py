"""TTTP / MTTKRP / Gram-matvec launch times (CUDA events, mean of 20 after 3
warm-ups) for the library selected by CPFIT_LIB: cfg 2 (fp64 and fp32, R=16),
a cfg 3-shaped Zipf instance (2e7 nnz, R=32) and a cfg 5-shaped order-4 fp32
instance (2e7 nnz, R=64).  Checks each MTTKRP against the default library's
result when CPFIT_REF_OUT is set (a .pt file written by a previous run)."""
import ctypes
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1910_02371_b200 as cp  # noqa: E402
from paper_1910_02371_b200 import _lib, synth  # noqa: E402

L = _lib.load()
s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def timeit(fn, n=20):
    for _ in range(3):
        fn()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / n


def case(name, t, F, dtype):
    code = 0 if dtype == torch.float64 else 1
    R = F[0].shape[1]
    pat = t.device_pattern()
    fp = _lib.ptr_array([f.data_ptr() for f in F])
    v = t.device_values(dtype)
    out = torch.empty(t.nnz, dtype=dtype, device="cuda")
    r = {"case": name}
    r["tttp_ms"] = timeit(lambda: _lib.check(L.cpfit_tttp(
        pat.handle, code, R, ctypes.c_void_p(v.data_ptr()), fp, ctypes.c_void_p(out.data_ptr()), s)))
    sums = [float(out.double().sum())]
    r["mttkrp_ms"] = []
    for m in range(t.order):
        sv = t.sorted_values(m, dtype)
        mo = torch.empty(t.shape[m], R, dtype=dtype, device="cuda")
        r["mttkrp_ms"].append(timeit(lambda: _lib.check(L.cpfit_mttkrp(
            pat.handle, m, code, R, ctypes.c_void_p(sv.data_ptr()), 1, fp,
            ctypes.c_void_p(mo.data_ptr()), s))))
        sums.append(float(mo.double().abs().sum()))
    r["checksums"] = sums
    print(json.dumps(r), flush=True)


which = sys.argv[1] if len(sys.argv) > 1 else "235"
if "2" in which:
    shape, keys, values, factors = synth.cfg2()
    t = cp.SparseTensor(shape, keys, values, validate=False)
    case("cfg2 f64 R16", t, [torch.from_numpy(f).cuda() for f in factors], torch.float64)
    case("cfg2 f32 R16", t, [torch.from_numpy(f).cuda().float() for f in factors], torch.float32)
    del t
if "3" in which:
    shape, keys, vals = synth.cfg3_device(nnz=20_000_000)
    t = cp.SparseTensor.from_device(shape, keys, vals)
    g = np.random.default_rng(0)
    F = [torch.from_numpy(g.random((d, 32)) / np.sqrt(32)).cuda() for d in shape]
    case("cfg3-like 2e7 f64 R32", t, F, torch.float64)
    del t
if "5" in which:
    shape, t, values, F = synth.cfg5_device(nnz=20_000_000)
    case("cfg5-like 2e7 f32 R64", t.with_values(values), F, torch.float32)
