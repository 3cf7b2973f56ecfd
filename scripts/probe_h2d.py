"""Is a numpy view of torch pinned memory seen as pinned, and what H2D
bandwidth do pinned / pageable copies reach on this box?"""
import time
import numpy as np
import torch

n = 2129264640 // 8
pinned = torch.empty(n, dtype=torch.float64, pin_memory=True)
pinned.numpy()[:] = 1.0
view = torch.from_numpy(pinned.numpy())
print("pinned.is_pinned", pinned.is_pinned(), "numpy view is_pinned", view.is_pinned())
dev = torch.empty(n, dtype=torch.float64, device="cuda")
for name, src in (("torch pinned", pinned), ("numpy view", view)):
    for _ in range(2):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        dev.copy_(src, non_blocking=True)
        t1 = time.perf_counter()
        torch.cuda.synchronize()
        t2 = time.perf_counter()
    print(f"{name}: enqueue {1e3*(t1-t0):.1f} ms, total {1e3*(t2-t0):.1f} ms, {n*8/(t2-t0)/1e9:.1f} GB/s")
pageable = np.ones(n)
pt = torch.from_numpy(pageable)
torch.cuda.synchronize()
t0 = time.perf_counter()
dev.copy_(pt, non_blocking=True)
torch.cuda.synchronize()
print(f"pageable: {n*8/(time.perf_counter()-t0)/1e9:.1f} GB/s")
