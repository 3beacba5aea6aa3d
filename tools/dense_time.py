"""Time the dense MTTKRP kernels (cfg 4: 800^3, R=64) per mode, fp64 DMMA and
TF32 tcgen05, the X.C GEMM, a CP-ALS sweep, and cuBLAS DGEMM as the FP64
denominator.  CUDA events on the launching stream."""
import json
import sys
import os

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_1910_02371_b200 import dense as DN


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


n = int(sys.argv[1]) if len(sys.argv) > 1 else 800
R = int(sys.argv[2]) if len(sys.argv) > 2 else 64
g = torch.Generator(device="cuda")
g.manual_seed(4)
X = torch.randn((n, n, n), generator=g, dtype=torch.float64, device="cuda")
F = [torch.randn((n, R), generator=g, dtype=torch.float64, device="cuda") for _ in range(3)]
flop = 2.0 * n ** 3 * R
out = {"n": n, "R": R}
out["f64_ms"] = [timed(lambda m=m: DN.dense_mttkrp(X, F, m)) for m in range(3)]
out["f64_tflops"] = [flop / (t * 1e-3) / 1e12 for t in out["f64_ms"]]
out["xc_ms"] = timed(lambda: DN.xc_product(X, F[2]))
Fs = [f.clone() for f in F]
out["als_sweep_ms"] = timed(lambda: DN.dense_als_sweep(X, Fs, 1e-5), reps=3)
T = DN.xc_product(X, F[2])
out["reduce_ms"] = [timed(lambda: DN.reduce_t(T, F[1], 1)), timed(lambda: DN.reduce_t(T, F[0], 0))]
out["gram_ms"] = timed(lambda: DN.gram_hadamard(F[:2]))
G = DN.gram_hadamard(F[:2])
M = DN.dense_mttkrp(X, F, 0)
out["solve_ms"] = timed(lambda: DN.solve_shared(G, M, 1e-5))
del T
a = torch.randn(8192, 8192, dtype=torch.float64, device="cuda")
pk = timed(lambda: a @ a)
out["cublas_dgemm_tflops"] = 2 * 8192 ** 3 / (pk * 1e-3) / 1e12
del a
out["f64_frac_of_dgemm"] = [t / out["cublas_dgemm_tflops"] for t in out["f64_tflops"]]
X32 = X.float()
del X
F32 = [f.float() for f in F]
out["tf32_ms"] = [timed(lambda m=m: DN.dense_mttkrp(X32, F32, m)) for m in range(3)]
out["tf32_hbm_gbs"] = [n ** 3 * 4 / (t * 1e-3) / 1e9 for t in out["tf32_ms"]]
out["tf32_xc_ms"] = timed(lambda: DN.xc_product(X32, F32[2]))
print(json.dumps(out))
