"""Per-step wall time of the streaming host API on c2 with pinned input."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2605_16058_b200 as sb
from paper_2605_16058_b200.configs import config2

a = config2(nlat=361, nlon=720, nt=1024, seed=0)
pinned = torch.empty(a.size, dtype=torch.float64, pin_memory=True)
pinned.numpy()[:] = a.reshape(-1, order="F")
host = sb.DenseTensor(pinned.numpy().reshape(a.shape, order="F"), copy=False)
ts = sb.TransformSet.build(a.shape, "dct")
for rep in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    ts_ = []
    for c in sb.tsvdm_tolerance_stream([host] * 5, ts, 1e-2):
        ts_.append(time.perf_counter() - t0)
    torch.cuda.synchronize()
    t = time.perf_counter() - t0
    print(f"rep {rep}: {[round(1e3*x) for x in ts_]} ms cumulative; {5 * a.size * 8 / t / 1e9:.1f} GB/s")
t0 = time.perf_counter()
for _ in range(3):
    c = sb.tsvdm_tolerance(host, ts, 1e-2)
print(f"plain host calls: {(time.perf_counter() - t0) / 3 * 1e3:.0f} ms per step")
