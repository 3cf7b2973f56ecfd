"""c3-shaped dense transform (1024 x 1024 x 512 f64, Haar-random 512 x 512 M):
forward mode-3 product on the DMMA GEMM kernel, timed with CUDA events
(3 warm-up, 10 timed).  Also the target for the ncu capture of
gemm_f64_kernel (DMMA pipe utilisation)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2605_16058_b200 as sb
from paper_2605_16058_b200.mode_product import forward_device
from paper_2605_16058_b200.transform_set import validate_transform

m, p, n = 1024, 1024, 512
rng = np.random.default_rng(0)
q, r = np.linalg.qr(rng.standard_normal((n, n)))
q = q * np.sign(np.diag(r))
ts = sb.TransformSet((validate_transform(np.asfortranarray(q)),))
dev = torch.device("cuda", 0)
x = sb.DeviceTensor(torch.randn(m * p * n, dtype=torch.float64, device=dev), (m, p, n))
for _ in range(3):
    forward_device(x, ts)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    forward_device(x, ts)
e1.record()
e1.synchronize()
ms = e0.elapsed_time(e1) / 10
flops = 2.0 * n * n * m * p
print(f"dense transform c3 shape: {ms:.3f} ms, {flops / ms / 1e9:.2f} TFLOP/s")
