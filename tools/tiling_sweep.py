"""Kernel-variant sweep: TTTP / MTTKRP time on BASELINE-like shapes for each
library build given on the command line (CPFIT_LIB per subprocess)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CASES = [
    ("cfg2_f64_R16", (10_000, 10_000, 10_000), 10_000_000, 16, "f64"),
    ("cfg3like_f64_R32", (480_189, 17_770, 2_182), 10_000_000, 32, "f64"),
    ("cfg1like_f64_R10", (2000, 2000, 2000), 10_000_000, 10, "f64"),
    ("cfg5like_f32_R64", (100_000, 100_000, 100_000, 1000), 10_000_000, 64, "f32"),
]

CHILD = r'''
import ctypes, json, sys, numpy as np, torch
sys.path.insert(0, ROOT)
import paper_1910_02371_b200 as cp
from paper_1910_02371_b200 import _lib, synth
name, shape, nnz, R, dt = json.loads(sys.argv[1])
rng = np.random.default_rng(1)
space = int(np.prod(np.array(shape, dtype=object)))
keys = synth.distinct_uniform_keys(rng, space, nnz)
t = cp.SparseTensor(tuple(shape), keys, rng.standard_normal(nnz), validate=False)
dtype = torch.float64 if dt == "f64" else torch.float32
code = 0 if dt == "f64" else 1
fs = [torch.randn(d, R, dtype=dtype, device="cuda") for d in shape]
L = _lib.load(); pat = t.device_pattern()
s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
vals = t.device_values(dtype); sv = [t.sorted_values(m, dtype) for m in range(len(shape))]
fp = _lib.ptr_array([f.data_ptr() for f in fs])
out = torch.empty(nnz, dtype=dtype, device="cuda")
mo = [torch.empty(d, R, dtype=dtype, device="cuda") for d in shape]
def timeit(fn, n=20):
    for _ in range(3): fn()
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n): fn()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / n
tt = timeit(lambda: _lib.check(L.cpfit_tttp(pat.handle, code, R, ctypes.c_void_p(vals.data_ptr()), fp, ctypes.c_void_p(out.data_ptr()), s)))
mt = [timeit(lambda m=m: _lib.check(L.cpfit_mttkrp(pat.handle, m, code, R, ctypes.c_void_p(sv[m].data_ptr()), 1, fp, ctypes.c_void_p(mo[m].data_ptr()), s))) for m in range(len(shape))]
chk = float(out.double().abs().sum()) + sum(float(m.double().abs().sum()) for m in mo)
print(json.dumps({"case": name, "tttp_ms": round(tt, 4), "mttkrp_ms": [round(x, 4) for x in mt], "checksum": chk}))
'''.replace("ROOT", repr(ROOT))

LIBS = sys.argv[1:] or [os.path.join(ROOT, "paper_1910_02371_b200", "libcpfit_b200.so")]
for case in CASES:
    for kv, lib in enumerate(LIBS):
        env = dict(os.environ, CPFIT_LIB=lib)
        r = subprocess.run([sys.executable, "-c", CHILD, json.dumps(case)], env=env,
                           capture_output=True, text=True)
        line = r.stdout.strip().splitlines()[-1] if r.stdout.strip() else r.stderr[-300:]
        print(f"{os.path.basename(lib)} {line}", flush=True)
