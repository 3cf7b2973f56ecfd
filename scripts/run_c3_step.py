"""Two c3 (1024x1024x512, Haar M, rank 32) fixed-rank compressions on a
device-resident input -- target for ncu launch lists."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2605_16058_b200 as sb
from paper_2605_16058_b200 import configs
from paper_2605_16058_b200.transform_set import validate_transform

a, mm = configs.config3()
ts = sb.TransformSet((validate_transform(mm),))
x = sb.DeviceTensor.from_host(sb.DenseTensor(a, copy=False), torch.device("cuda", 0))
for _ in range(2):
    c = sb.tsvdm_fixed_rank(x, ts, 32)
torch.cuda.synchronize()
print("ok", c.factors.total_rank)
