"""Timing of the pieces of compress.prune_refine on c2 (CUDA events)."""
import sys, time
import numpy as np, torch
sys.path.insert(0, ".")
import paper_2605_16058_b200 as sb
from paper_2605_16058_b200 import compress as cp, _native as nat
from paper_2605_16058_b200.configs import config2
from paper_2605_16058_b200.mode_product import forward_device

a = config2(nlat=361, nlon=720, nt=1024, seed=0)
ts = sb.TransformSet.build(a.shape, "dct")
x = sb.DeviceTensor.from_host(sb.DenseTensor(a, copy=False), torch.device("cuda", 0))
ah = forward_device(x, ts)
m, p, n = a.shape
dev = ah.device
def t(fn, reps=20):
    fn(); torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(reps): fn()
    torch.cuda.synchronize(); return (time.perf_counter() - t0) / reps * 1e3
f_dev = torch.empty(n, dtype=torch.float64, device=dev)
def energy():
    nat.call("starm_slice_energy_f64", ah.data.data_ptr(), m * p, n, f_dev.data_ptr(), nat.stream_ptr(dev))
print("energy kernel", t(energy))
f = f_dev.cpu().numpy()
print("energy + D2H", t(lambda: (energy(), f_dev.cpu())))
sel = cp.prune_choose(f, 1e-2)
print("choose (host)", t(lambda: cp.prune_choose(f, 1e-2)))
print("refine", t(lambda: cp.prune_refine(ah, f, 1e-2, sel)))
print("plan", t(lambda: cp.prune_plan(ah, 1e-2)))
r = cp.prune_refine(ah, f, 1e-2, sel)
print("kept", sel[0].size, "->", r[0].size)
