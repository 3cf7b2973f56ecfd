"""Run the c2 values pass (bidiagonal path) twice -- target for ncu launch lists."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2605_16058_b200 as sb
from paper_2605_16058_b200.configs import config2
from paper_2605_16058_b200.mode_product import forward_device
from paper_2605_16058_b200.slice_svd import svd_values_device

nt = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
a = config2(nlat=361, nlon=720, nt=nt, seed=0)
ts = sb.TransformSet.build(a.shape, "dct")
x = sb.DeviceTensor.from_host(sb.DenseTensor(a, copy=False), torch.device("cuda", 0))
ahat = forward_device(x, ts)
for _ in range(2):
    s = svd_values_device(sb.DeviceTensor(ahat.data, a.shape))
torch.cuda.synchronize()
print("ok", float(s.max()))
