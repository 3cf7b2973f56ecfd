"""Full-size run of one BASELINE config on cuda:0 through the public API:
time the compression (device-resident input) and check the realised error
against the energy identity  relerr^2 = discarded / total  (orthogonal M).

usage: python scripts/run_config.py c3 [reps]
"""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2605_16058_b200 as sb
from paper_2605_16058_b200 import configs
from paper_2605_16058_b200.compress import reconstruct_device, relative_error_device
from paper_2605_16058_b200.transform_set import validate_transform

name = sys.argv[1]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
dev = torch.device("cuda", 0)
t0 = time.time()
if name == "c1":
    a = configs.config1()
    ts = sb.TransformSet.build(a.shape, "dct")
    run = lambda x: sb.tsvdm_fixed_rank(x, ts, 10)
elif name == "c2":
    a = configs.config2()
    ts = sb.TransformSet.build(a.shape, "dct")
    run = lambda x: sb.tsvdm_tolerance(x, ts, 1e-2)
elif name == "c3":
    a, mm = configs.config3()
    ts = sb.TransformSet((validate_transform(mm),))
    run = lambda x: sb.tsvdm_fixed_rank(x, ts, 32)
elif name == "c5":
    ahat, mm = configs.config5_transform_domain()
    ts = sb.TransformSet((validate_transform(mm),))
    # original-domain tensor = ahat x_3 M^T, formed on the device
    xh = sb.DeviceTensor.from_host(sb.DenseTensor(ahat, copy=False), dev)
    del ahat
    from paper_2605_16058_b200.mode_product import inverse_device
    a = None
    xdev = inverse_device(xh, ts)
    del xh
    run = lambda x: sb.tsvdm_fixed_rank(x, ts, 16)
    if len(sys.argv) > 3 and sys.argv[3] == "tol":
        run = lambda x: sb.tsvdm_tolerance(x, ts, 1e-4)
else:
    raise SystemExit(f"unknown config {name}")
if a is not None:
    xdev = sb.DeviceTensor.from_host(sb.DenseTensor(a, copy=False), dev)
    del a
print(f"{name}: dims {xdev.dims}, setup {time.time() - t0:.1f}s", flush=True)
for i in range(reps):
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    c = run(xdev)
    e1.record()
    e1.synchronize()
    ms = e0.elapsed_time(e1)
    print(f"  rep {i}: {ms:.1f} ms  total_rank {c.factors.total_rank}", flush=True)
rec = reconstruct_device(c, dev)
err = relative_error_device(xdev, rec)
pred = float(np.sqrt(c.discarded_energy / c.total_energy))
print(f"  realised relerr {err:.10g}  predicted {pred:.10g}  diff {abs(err - pred):.3g}")
ok = abs(err - pred) <= 1e-8 + 1e-6 * pred
print("OK" if ok else "MISMATCH")
sys.exit(0 if ok else 1)
