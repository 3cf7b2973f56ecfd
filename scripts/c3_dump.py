"""Full-size c3 on cuda:0 through the public API: fixed-rank (32) t-SVDM
energies and every slice's singular values -> gpurun_out/c3_gpu.npz, for
tests/fullsize_c3_parity.py."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2605_16058_b200 as sb
from paper_2605_16058_b200.configs import config3
from paper_2605_16058_b200.transform_set import validate_transform

a, mm = config3()
ts = sb.TransformSet((validate_transform(mm),))
x = sb.DeviceTensor.from_host(sb.DenseTensor(a, copy=False), torch.device("cuda", 0))
c = sb.tsvdm_fixed_rank(x, ts, 32)
s = sb.svd_values_only(sb.to_transform_domain(x, ts))
os.makedirs("gpurun_out", exist_ok=True)
np.savez("gpurun_out/c3_gpu.npz", s=s.cpu().numpy(), discarded=c.discarded_energy,
         total=c.total_energy)
print("dumped", c.relative_error())
