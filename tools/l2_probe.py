"""L2 read-bandwidth probe sweep: buffer size x resident CTAs per SM
(cpfit_probe_l2_read; CUDA events)."""
import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_1910_02371_b200 import _lib

L = _lib.load()
sms = torch.cuda.get_device_properties(0).multi_processor_count
s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
res = {}
for mb in (16, 32, 48, 64, 96):
    buf = torch.ones(mb << 20, dtype=torch.uint8, device="cuda")
    for per_sm in (1, 2, 4):
        out = torch.empty(sms * per_sm * 512, dtype=torch.int32, device="cuda")

        def run(reps):
            _lib.check(L.cpfit_probe_l2_read(ctypes.c_void_p(buf.data_ptr()), buf.numel(), reps,
                                             ctypes.c_void_p(out.data_ptr()), out.numel(), s))
        run(3)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        run(20)
        b.record()
        torch.cuda.synchronize()
        res[f"{mb}MB_x{per_sm}"] = round(buf.numel() * 20 / (a.elapsed_time(b) * 1e-3) / 1e9)
print(json.dumps(res))
