"""Where does the e2e streaming path lose time vs the device-resident step?"""
import sys, time
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_2605_16058_b200 as sb
from paper_2605_16058_b200.configs import config2

a = config2(nlat=361, nlon=720, nt=1024, seed=0)
pinned = torch.empty(a.size, dtype=torch.float64, pin_memory=True)
pinned.numpy()[:] = a.reshape(-1, order="F")
host = sb.DenseTensor(pinned.numpy().reshape(a.shape, order="F"), copy=False)
src = torch.from_numpy(np.ascontiguousarray(host.data))
print("from_numpy view pinned:", src.is_pinned(), "same ptr:", src.data_ptr() == pinned.data_ptr())
ts = sb.TransformSet.build(a.shape, "dct")
dev = torch.device("cuda", 0)
# H2D alone
buf = torch.empty(a.size, dtype=torch.float64, device=dev)
for p in (pinned, src):
    torch.cuda.synchronize(); t0 = time.perf_counter(); buf.copy_(p, non_blocking=True); t1 = time.perf_counter(); torch.cuda.synchronize(); t2 = time.perf_counter()
    print(f"h2d: call {1e3*(t1-t0):.1f} ms, total {1e3*(t2-t0):.1f} ms ({a.size*8/(t2-t0)/1e9:.1f} GB/s)")
for _ in sb.tsvdm_tolerance_stream([host] * 2, ts, 1e-2):
    pass
torch.cuda.synchronize()
t0 = time.perf_counter(); marks = []
for ch in sb.tsvdm_tolerance_stream([host] * 6, ts, 1e-2):
    marks.append(time.perf_counter())
torch.cuda.synchronize()
print("per-item ms:", [round(1e3 * (b - a_), 1) for a_, b in zip([t0] + marks[:-1], marks)])
x = sb.DeviceTensor.from_host(host, dev)
torch.cuda.synchronize(); t0 = time.perf_counter()
for _ in range(6):
    c = sb.tsvdm_tolerance(x, ts, 1e-2); h = c.to_host()
torch.cuda.synchronize(); print("device-resident + to_host per step ms:", round(1e3 * (time.perf_counter() - t0) / 6, 1))
