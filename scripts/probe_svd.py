"""SVD kernel probe: timing + per-phase counters on c2-like slices for a few
tuning settings, plus an accuracy check against LAPACK on a subset."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import oracle  # checker only
import paper_2605_16058_b200 as sb
from paper_2605_16058_b200 import _native as nat
from paper_2605_16058_b200.configs import config2, dct_matrix_np
from paper_2605_16058_b200.slice_svd import svd_values_device

dev = torch.device("cuda", 0)
lib = nat.load()
a = config2(nlat=361, nlon=720, nt=64, seed=0)
ahat = oracle.ttm(a, 2, dct_matrix_np(64))
m, p, n = ahat.shape
x = sb.DeviceTensor.from_host(sb.DenseTensor(ahat), dev)
ref = oracle.svd_values_only(ahat, indices=range(0, n, 8))


def run(tag, inner, qr):
    lib.starm_svd_tune(inner, -1, qr, 1)
    nat.svd_stats(reset=True)
    s = svd_values_device(x)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    nat.svd_stats(reset=True)
    e0.record()
    s = svd_values_device(x)
    e1.record()
    e1.synchronize()
    st = nat.svd_stats(reset=True)
    sh = s.cpu().numpy().reshape((min(m, p), n), order="F")
    worst = 0.0
    for i in range(0, n, 8):
        r = ref[:, i]
        tol = 1e-10 * r + 64 * 2.2e-16 * r[0]
        worst = max(worst, float(np.max(np.abs(sh[:, i] - r) / tol)))
    out = dict(tag=tag, ms=e0.elapsed_time(e1), worst_over_tol=worst,
               sweeps_per_slice=st["sweeps"] / max(st["slices"], 1),
               rot_frac=st["rotated"] / max(st["pairs"], 1))
    tot = sum(st[k] for k in ("cyc_gram", "cyc_eig", "cyc_apply", "cyc_qr", "cyc_final", "cyc_load"))
    for k in ("cyc_gram", "cyc_eig", "cyc_apply", "cyc_qr", "cyc_final", "cyc_load"):
        out[k] = round(st[k] / max(tot, 1), 3)
    out["Mcyc_per_slice"] = tot / max(st["slices"], 1) / 1e6
    print(json.dumps(out), flush=True)


for inner in (1, 2, 6):
    for qr in (0, 1):
        run(f"inner{inner}_qr{qr}", inner, qr)
lib.starm_svd_tune(1, -1, 1, 0)
