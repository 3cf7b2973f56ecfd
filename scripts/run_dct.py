"""c2 forward DCT (the transform launch) twice: target for ncu captures."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2605_16058_b200 as sb
from paper_2605_16058_b200.configs import config2
from paper_2605_16058_b200.mode_product import forward_device

a = config2(nlat=361, nlon=720, nt=1024, seed=0)
ts = sb.TransformSet.build(a.shape, "dct")
x = sb.DeviceTensor.from_host(sb.DenseTensor(a, copy=False), torch.device("cuda", 0))
for _ in range(3):
    forward_device(x, ts)
torch.cuda.synchronize()
print("ok")
