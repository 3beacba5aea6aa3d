"""One cuBLAS DGEMM (torch float64 matmul), for an ncu look at its launch shape."""
import torch
a = torch.randn(8192, 8192, dtype=torch.float64, device="cuda")
for _ in range(2):
    a @ a
torch.cuda.synchronize()
print("ok")
