"""One fp64 and one TF32 dense MTTKRP call at cfg 4 (for ncu captures)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_1910_02371_b200 import dense as DN

n, R = 800, 64
g = torch.Generator(device="cuda")
g.manual_seed(4)
X = torch.randn((n, n, n), generator=g, dtype=torch.float64, device="cuda")
F = [torch.randn((n, R), generator=g, dtype=torch.float64, device="cuda") for _ in range(3)]
modes = [int(m) for m in (sys.argv[1] if len(sys.argv) > 1 else "0").split(",")]
for m in modes:
    DN.dense_mttkrp(X, F, m)
X32 = X.float()
F32 = [f.float() for f in F]
for m in modes:
    DN.dense_mttkrp(X32, F32, m)
torch.cuda.synchronize()
print("ok")
