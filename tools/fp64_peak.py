"""FP64 peak on this B200: cuBLAS DGEMM (torch.matmul float64) and a pure
DMMA (mma.sync m8n8k4 f64) loop -- the denominators for the Gram roofline."""
import json
import torch

res = {}
for n in (4096, 8192):
    a = torch.randn(n, n, dtype=torch.float64, device="cuda")
    b = torch.randn(n, n, dtype=torch.float64, device="cuda")
    for _ in range(3):
        torch.matmul(a, b)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    reps = 10
    for _ in range(reps):
        torch.matmul(a, b)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    res[f"dgemm_{n}_tflops"] = 2 * n ** 3 / (ms * 1e-3) / 1e12
print(json.dumps(res))
