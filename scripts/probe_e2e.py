"""Where the c2 drop-in host call (tsvdm_tolerance(DenseTensor)) spends its
time: plain H2D, block-wise 2-D H2D alone, block-wise upload + transform,
the whole call; for several block counts."""
import sys, time
import numpy as np, torch
sys.path.insert(0, ".")
import paper_2605_16058_b200 as sb
from paper_2605_16058_b200 import _native as nat, mode_product as mp
from paper_2605_16058_b200.configs import config2

dev = torch.device("cuda", 0)
a = config2(nlat=361, nlon=720, nt=1024, seed=0)
m, p, n = a.shape
pinned = torch.empty(a.size, dtype=torch.float64, pin_memory=True)
pinned.numpy()[:] = a.reshape(-1, order="F")
host = sb.DenseTensor(pinned.numpy().reshape(a.shape, order="F"), copy=False)
ts = sb.TransformSet.build(a.shape, "dct")
x = torch.empty(a.size, dtype=torch.float64, device=dev)

def timed(fn, reps=5):
    fn(); torch.cuda.synchronize()
    ts_ = []
    for _ in range(reps):
        torch.cuda.synchronize(); t0 = time.perf_counter(); fn(); torch.cuda.synchronize()
        ts_.append((time.perf_counter() - t0) * 1e3)
    return min(ts_), sorted(ts_)[len(ts_) // 2]

print("plain H2D", timed(lambda: x.copy_(pinned, non_blocking=True)))
rows = m * p
for nb in (4, 8, 16, 32, 64):
    step = max(128, -(-rows // nb + 127) // 128 * 128)
    def c2d():
        h = nat.stream_ptr(dev)
        for f0 in range(0, rows, step):
            nf = min(step, rows - f0)
            nat.call("starm_copy2d_h2d", x.data_ptr() + 8 * f0, 8 * rows, pinned.data_ptr() + 8 * f0, 8 * rows, 8 * nf, n, h)
    print("2-D H2D blocks", nb, timed(c2d))
    print("   from_host  ", nb, timed(lambda: mp.DeferredResidual.from_host(host, ts[0], dev, blocks=nb)))
    mp.PIPELINE_BLOCKS = nb
    print("   whole call ", nb, timed(lambda: sb.tsvdm_tolerance(host, ts, 1e-2)))
xd = sb.DeviceTensor(x, a.shape)
print("device-resident call", timed(lambda: sb.tsvdm_tolerance(xd, ts, 1e-2)))
import os
os.environ["STARM_PIPELINE"] = "0"
print("whole call, one-shot upload", timed(lambda: sb.tsvdm_tolerance(host, ts, 1e-2)))
