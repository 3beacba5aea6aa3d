import time, torch, numpy as np
n = 10_000_000
cs = torch.cuda.Stream()
dv = torch.empty(n, dtype=torch.float64, device="cuda")
hp = torch.empty(n, dtype=torch.float64, pin_memory=True)
f = torch.randn(10000, 16, dtype=torch.float64).pin_memory()
fn = f.numpy()
x = torch.empty(1000, device="cuda")
def during(fn_, label):
    rows = []
    for _ in range(5):
        torch.cuda.synchronize()
        with torch.cuda.stream(cs):
            hp.copy_(dv, non_blocking=True)
        a = time.perf_counter(); fn_(); b = time.perf_counter()
        torch.cuda.synchronize(); rows.append((b - a) * 1e3)
    print(label, round(float(np.median(rows)), 3))
during(lambda: torch.from_numpy(fn).to("cuda"), "h2d from pinned-backed numpy (blocking)")
during(lambda: torch.from_numpy(fn).to("cuda", non_blocking=True), "h2d non_blocking")
during(lambda: (x.add_(1), torch.cuda.current_stream().synchronize()), "kernel + stream sync")
hs = torch.empty(1000, pin_memory=True)
during(lambda: hs.copy_(x), "small d2h torch copy")
during(lambda: torch.empty(160000, dtype=torch.float64, pin_memory=True), "pinned alloc")
print("is_pinned", torch.from_numpy(fn).is_pinned())
