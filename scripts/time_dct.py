"""Time the c2 forward and inverse DCT launches (CUDA events, 10 reps)."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2605_16058_b200 as sb
from paper_2605_16058_b200.configs import config2
from paper_2605_16058_b200.mode_product import forward_device, inverse_device

a = config2(nlat=361, nlon=720, nt=1024, seed=0)
ts = sb.TransformSet.build(a.shape, "dct")
x = sb.DeviceTensor.from_host(sb.DenseTensor(a, copy=False), torch.device("cuda", 0))
for name, fn in (("forward", forward_device), ("inverse", inverse_device)):
    for _ in range(3):
        fn(x, ts)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(10):
        fn(x, ts)
    e1.record()
    e1.synchronize()
    ms = e0.elapsed_time(e1) / 10
    print(f"{name}: {ms:.3f} ms, {2 * a.size * 8 / ms / 1e6:.0f} GB/s")
