"""SVD kernel probe: timing + per-phase counters on c2-like slices for the
bidiagonal values path and the Jacobi path, plus accuracy vs LAPACK."""
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
nt = int(sys.argv[1]) if len(sys.argv) > 1 else 64
a = config2(nlat=361, nlon=720, nt=nt, seed=0)
ahat = oracle.ttm(a, 2, dct_matrix_np(nt))
m, p, n = ahat.shape
x = sb.DeviceTensor.from_host(sb.DenseTensor(ahat), dev)
step = max(1, n // 8)
ref = oracle.svd_values_only(ahat, indices=range(0, n, step))


def run(tag, inner, mode):
    lib.starm_svd_tune(inner, -1, mode, 1)
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
    worst, worst_abs = 0.0, 0.0
    for i in range(0, n, step):
        r = ref[:, i]
        tol = 1e-10 * r + 64 * 2.2e-16 * r[0]
        worst = max(worst, float(np.max(np.abs(sh[:, i] - r) / tol)))
        worst_abs = max(worst_abs, float(np.max(np.abs(sh[:, i] - r)) / r[0]))
    out = dict(tag=tag, ms=e0.elapsed_time(e1), worst_over_tol=worst, worst_abs_rel_smax=worst_abs)
    cyc = {k: v for k, v in st.items() if k.startswith("cyc_")}
    tot = sum(cyc.values())
    for k, v in cyc.items():
        out[k] = round(v / max(tot, 1), 3)
    out["sweeps_per_slice"] = st["sweeps"] / max(st["slices"], 1)
    print(json.dumps(out), flush=True)


run("bidiag", 1, 1)
run("jacobi_inner1", 1, 0)
lib.starm_svd_tune(1, -1, 1, 0)
