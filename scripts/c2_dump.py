"""Full-size c2 on cuda:0 through the public API: tolerance t-SVDM result and
every slice's singular values -> gpurun_out/c2_gpu.npz, for the CPU parity
check tests/fullsize_c2_parity.py (run where the oracle is)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2605_16058_b200 as sb
from paper_2605_16058_b200.configs import config2

a = config2(nlat=361, nlon=720, nt=1024, seed=0)
ts = sb.TransformSet.build(a.shape, "dct")
dev = torch.device("cuda", 0)
x = sb.DeviceTensor.from_host(sb.DenseTensor(a, copy=False), dev)
c = sb.tsvdm_tolerance(x, ts, 1e-2)
s = sb.svd_values_only(sb.to_transform_domain(x, ts))
ranks = np.asarray(c.ranks)
os.makedirs("gpurun_out", exist_ok=True)
f = c.factors.to_host()
np.savez("gpurun_out/c2_gpu.npz", s=s.cpu().numpy(), ranks=np.asarray(ranks),
         discarded=c.discarded_energy, total=c.total_energy, u_data=f.u_data, g_data=f.g_data)
print("dumped", int(np.sum(ranks)), c.relative_error())
