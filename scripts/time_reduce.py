"""Time the c2 values pass stopped after svd_reduce_kernel (tune mode 3) with
CUDA events; prints ms per launch."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2605_16058_b200 as sb
from paper_2605_16058_b200 import _native as nat
from paper_2605_16058_b200.configs import config2
from paper_2605_16058_b200.mode_product import forward_device
from paper_2605_16058_b200.slice_svd import svd_values_device

a = config2(nlat=361, nlon=720, nt=1024, seed=0)
ts = sb.TransformSet.build(a.shape, "dct")
x = sb.DeviceTensor.from_host(sb.DenseTensor(a, copy=False), torch.device("cuda", 0))
ah = sb.DeviceTensor(forward_device(x, ts).data, a.shape)
s_ref = svd_values_device(ah)
nat.load().starm_svd_tune(-1, -1, 3, -1)
svd_values_device(ah)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(3):
    svd_values_device(ah)
e1.record()
e1.synchronize()
print("reduce ms", e0.elapsed_time(e1) / 3)
