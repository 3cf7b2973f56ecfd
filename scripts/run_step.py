"""One warm + one measured c2 compression step (device-resident input) --
target for ncu launch lists / captures."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2605_16058_b200 as sb
from paper_2605_16058_b200.configs import config2

nt = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
if len(sys.argv) > 2:  # svd path mode (starm_svd_tune), e.g. 2 = bulge window in global memory
    from paper_2605_16058_b200 import _native as nat
    nat.load().starm_svd_tune(-1, -1, int(sys.argv[2]), -1)
a = config2(nlat=361, nlon=720, nt=nt, seed=0)
ts = sb.TransformSet.build(a.shape, "dct")
x = sb.DeviceTensor.from_host(sb.DenseTensor(a, copy=False), torch.device("cuda", 0))
for _ in range(2):
    c = sb.tsvdm_tolerance(x, ts, 1e-2)
torch.cuda.synchronize()
print("ok", c.factors.total_rank, c.relative_error())
