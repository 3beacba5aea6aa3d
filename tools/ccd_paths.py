"""Per-(path, mode) timing of one CCD++ column step at the cfg 3 shape
(CUDA events).  usage: python tools/ccd_paths.py [nnz]"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1910_02371_b200 as cp  # noqa: E402
from paper_1910_02371_b200 import _lib, synth  # noqa: E402
from paper_1910_02371_b200.losses import tttp_affine  # noqa: E402
from paper_1910_02371_b200.optim import _ccd_col_ptrs, _stream  # noqa: E402

nnz = int(sys.argv[1]) if len(sys.argv) > 1 else 100_480_507
shape, keys, vals = synth.cfg3_device(nnz=nnz)
t = cp.SparseTensor.from_device(shape, keys, vals)
g = np.random.default_rng(0)
F = [torch.from_numpy(g.random((d, 2)) / np.sqrt(2)).cuda() for d in shape]
L = _lib.load()
pat = t.device_pattern()
cols = [f.t().contiguous() for f in F]
rhat = tttp_affine(t, F, -1.0, 1.0, torch.float64)
keep, ptrs = _ccd_col_ptrs(cols, 0)
for path in ("task", "flat", "priv"):
    os.environ["CPFIT_CCD_PATH"] = path
    for mode in range(3):
        for fold in ((1, 0) if mode == 0 else (0,)):
            def call():
                _lib.check(L.cpfit_ccd_step(pat.handle, mode, ptrs,
                                            ctypes.c_void_p(rhat.data_ptr()), fold, None, 1e-5,
                                            None, _stream()), "ccd_step")
            try:
                call()
            except Exception as e:  # noqa: BLE001
                print(path, mode, fold, "n/a", e)
                continue
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(5):
                call()
            e1.record()
            torch.cuda.synchronize()
            print(f"path={path} mode={mode} fold={fold}: {e0.elapsed_time(e1) / 5:.3f} ms")
