"""Bitwise determinism of the values pass (plain vs state-keeping, repeated)."""
import sys
import numpy as np
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
ah = sb.DeviceTensor(forward_device(x, ts).data, a.shape)
outs = []
for keep in (False, True, False, True):
    r = svd_values_device(ah, keep_state=keep)
    s = r[0] if keep else r
    outs.append(s.cpu().numpy())
for i in range(1, 4):
    d = outs[i] != outs[0]
    print(i, "mismatches", int(d.sum()), "max rel", float(np.max(np.abs(outs[i] - outs[0]) / np.maximum(outs[0], 1e-300))))
