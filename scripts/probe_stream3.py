"""c2 through tsvdm_tolerance_stream (H2D of tensor k+1 behind tensor k): per-tensor ms."""
import sys, time, os
import numpy as np, torch
sys.path.insert(0, ".")
import paper_2605_16058_b200 as sb
from paper_2605_16058_b200.configs import config2
a = config2(nlat=361, nlon=720, nt=1024, seed=0)
pinned = torch.empty(a.size, dtype=torch.float64, pin_memory=True)
pinned.numpy()[:] = a.reshape(-1, order="F")
host = sb.DenseTensor(pinned.numpy().reshape(a.shape, order="F"), copy=False)
ts = sb.TransformSet.build(a.shape, "dct")
for _ in sb.tsvdm_tolerance_stream([host] * 2, ts, 1e-2): pass
torch.cuda.synchronize(); t0 = time.perf_counter()
for _ in sb.tsvdm_tolerance_stream([host] * 8, ts, 1e-2): pass
torch.cuda.synchronize(); print(os.environ.get("TAG", ""), "stream ms/tensor", (time.perf_counter() - t0) / 8 * 1e3)
