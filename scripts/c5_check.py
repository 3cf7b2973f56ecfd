"""Full-size c5 against its analytic golden: every slice of the M-domain
tensor is U_i diag(0.8^j) V_i^T, so after A = Ahat x_3 M^T (on the device)
the t-SVDM must return sigma_j = 0.8^j in every slice, and the fixed-rank-16
energies are closed-form.  Prints the deviations (run under gpurun)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2605_16058_b200 as sb
from paper_2605_16058_b200 import configs
from paper_2605_16058_b200.mode_product import inverse_device
from paper_2605_16058_b200.transform_set import validate_transform

dev = torch.device("cuda", 0)
ahat, mm = configs.config5_transform_domain()
ts = sb.TransformSet((validate_transform(mm),))
xh = sb.DeviceTensor.from_host(sb.DenseTensor(ahat, copy=False), dev)
del ahat
x = inverse_device(xh, ts)
del xh
s = sb.svd_values_only(sb.to_transform_domain(x, ts)).cpu().numpy()  # (64, 4096)
gold = 0.8 ** np.arange(64)
dev_abs = np.max(np.abs(s - gold[:, None]))
dev_rel = np.max(np.abs(s - gold[:, None]) / gold[:, None])
c = sb.tsvdm_fixed_rank(x, ts, 16)
tot = 4096 * np.sum(gold ** 2)
disc = 4096 * np.sum(gold[16:] ** 2)
print(f"c5 full size (8192x64x4096, Haar M): sigma vs 0.8^j: max abs {dev_abs:.3e}, max rel {dev_rel:.3e} "
      f"(sigma_63 = {gold[63]:.3e})")
print(f"fixed rank 16: relative error {c.relative_error():.12g} vs analytic {np.sqrt(disc / tot):.12g}; "
      f"total energy rel diff {abs(c.total_energy - tot) / tot:.3e}")
