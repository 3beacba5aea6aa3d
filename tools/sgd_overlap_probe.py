"""Does sampling step k+1 on a side stream (helper thread) overlap with step k's
TTTP / sorts / MTTKRPs?  cfg 5 scale; prints serial vs pipelined ms per step."""
import concurrent.futures as cf
import ctypes
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1910_02371_b200 as cp  # noqa: E402
from paper_1910_02371_b200 import _lib, synth  # noqa: E402
from paper_1910_02371_b200.core import _dtype_code  # noqa: E402
from paper_1910_02371_b200.losses import tttp_affine  # noqa: E402
from paper_1910_02371_b200.optim import (SolverConfig, _ptrs, _sgd_apply_device, _sgd_ls_device,  # noqa: E402
                                          _stream)
from paper_1910_02371_b200.sampling import sample_tensor  # noqa: E402

nnz = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000_000
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 8
shape, tn, values, F = synth.cfg5_device(nnz=nnz)
t = tn.with_values(values)
cfg = SolverConfig(rank=64, algorithm="sgd", step=1e-3, reg=1e-4, sample_rate=0.01)
dtype = torch.float32
L = _lib.load()
root = cp.RngState(5).child(1)

# serial reference
Fs = [f.clone() for f in F]
for it in range(2):
    _sgd_ls_device(t, Fs, cfg, root.child(it))
torch.cuda.synchronize()
t0 = time.perf_counter()
for it in range(2, 2 + steps):
    _sgd_ls_device(t, Fs, cfg, root.child(it))
torch.cuda.synchronize()
serial = (time.perf_counter() - t0) / steps * 1e3

side = torch.cuda.Stream()
main = torch.cuda.current_stream()
pool = cf.ThreadPoolExecutor(max_workers=1)


def prefetch(it):
    torch.cuda.set_device(0)
    with torch.cuda.stream(side):
        s = sample_tensor(t, cfg.sample_rate, root.child(it), dtype)
        s.device_values(dtype).record_stream(main)
        ev = torch.cuda.Event()
        ev.record(side)
    return s, ev


def consume(Fp, sampled, ev):
    main.wait_event(ev)
    phi1 = tttp_affine(sampled, Fp, 2.0, -2.0, dtype)
    pat = sampled.device_pattern()
    grads = []
    for mode in range(t.order):
        g = torch.empty((t.shape[mode], 64), dtype=dtype, device=Fp[0].device)
        _lib.check(L.cpfit_mttkrp(pat.handle, mode, _dtype_code(dtype), 64,
                                  ctypes.c_void_p(phi1.data_ptr()), 0, _ptrs(Fp),
                                  ctypes.c_void_p(g.data_ptr()), _stream()), "mttkrp")
        grads.append(g)
    shrink = 2.0 * cfg.step * cfg.reg * cfg.sample_rate
    _sgd_apply_device(Fp, grads, cfg.step, shrink, check=False)


Fp = [f.clone() for f in F]
fut = pool.submit(prefetch, 0)
keep = []
for it in range(2):
    s, ev = fut.result()
    fut = pool.submit(prefetch, it + 1)
    consume(Fp, s, ev)
    keep.append(s)
torch.cuda.synchronize()
t0 = time.perf_counter()
for it in range(2, 2 + steps):
    s, ev = fut.result()
    fut = pool.submit(prefetch, it + 1)
    consume(Fp, s, ev)
    keep.append(s)
torch.cuda.synchronize()
piped = (time.perf_counter() - t0) / steps * 1e3
fut.result()
torch.cuda.synchronize()
err = max(float((a - b).abs().max()) for a, b in zip(Fs, Fp))
print(f"serial {serial:.2f} ms/step, pipelined {piped:.2f} ms/step, max |dF| serial vs pipelined {err:.3e}")
