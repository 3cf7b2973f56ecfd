"""Full-size c4 on cuda:0 (SURVEY 8c restatement: f32 upcast, raw M): every
slice's singular values, the device threshold's ranks and energies ->
gpurun_out/c4_gpu.npz, for tests/fullsize_c4_parity.py."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2605_16058_b200 as sb
from paper_2605_16058_b200.configs import config4

a32, mm, _ = config4()
x = sb.DeviceTensor.from_host(sb.DenseTensor(np.asfortranarray(a32, dtype=np.float64), copy=False),
                              torch.device("cuda", 0))
del a32
ahat = sb.ttm(x, 2, mm)
s = sb.svd_values_only(ahat)
th = sb.compute_threshold(s, 1e-3)
os.makedirs("gpurun_out", exist_ok=True)
np.savez("gpurun_out/c4_gpu.npz", s=s.cpu().numpy(), ranks=th.ranks.cpu().numpy(), j=th.j, tau=th.tau,
         discarded=th.discarded_energy, total=th.total_energy)
print("dumped", int(th.ranks.sum()))
