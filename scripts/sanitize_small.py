"""Small end-to-end workload for compute-sanitizer (memcheck / racecheck):
every kernel family once on tiny shapes -- DCT + tcgen05 residual (n = 256),
dense DMMA TTM, values / full / truncated SVD (QR + band + bulge + bisection
+ vectors), threshold, fused reconstruction + error."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2605_16058_b200 as sb

rng = np.random.default_rng(0)
a = np.asfortranarray(rng.standard_normal((24, 40, 256)))
a += np.einsum("i,j,k->ijk", rng.standard_normal(24), rng.standard_normal(40), rng.standard_normal(256))
t = sb.DenseTensor(a)
ts = sb.TransformSet.build(a.shape, "dct")
c = sb.tsvdm_tolerance(t, ts, 0.2)
x = sb.DeviceTensor.from_host(t)
rec, err = sb.reconstruct_fused(sb.tsvdm_tolerance(x, ts, 0.2), a=x)
q, r = np.linalg.qr(rng.standard_normal((12, 12)))
b = np.asfortranarray(rng.standard_normal((70, 33, 12)))
ts2 = sb.TransformSet((sb.validate_transform(q * np.sign(np.diag(r))),))
f = sb.tsvdm_fixed_rank(sb.DenseTensor(b), ts2, 5)
full = sb.svd_all_slices(sb.DenseTensor(b))
tall = sb.svd_values_only(sb.DenseTensor(np.asfortranarray(rng.standard_normal((1500, 20, 2)))))
torch.cuda.synchronize()
print("sanitize workload ok", int(c.ranks.sum()), err, f.factors.total_rank, full.s.shape, tall.shape)
