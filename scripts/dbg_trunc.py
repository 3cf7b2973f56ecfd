"""Per-slice check of the truncated factors: ||A_i - U_i G_i||_F^2 against
the LAPACK tail energy sum_{j>=k} sigma_j^2, on config3-shaped slices.

usage: python scripts/dbg_trunc.py [nx] [nt] [rank]
"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import oracle  # checker only
import paper_2605_16058_b200 as sb
from paper_2605_16058_b200 import configs
from paper_2605_16058_b200.slice_svd import svd_truncated_device

nx = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
nt = int(sys.argv[2]) if len(sys.argv) > 2 else 8
k = int(sys.argv[3]) if len(sys.argv) > 3 else 32
dev = torch.device("cuda", 0)
a, mm = configs.config3(nx=nx, ny=nx, nt=nt)
ahat = oracle.ttm(a, 2, mm)
m, p, n = ahat.shape
x = sb.DeviceTensor.from_host(sb.DenseTensor(ahat), dev)
ranks = torch.full((n,), k, dtype=torch.int64, device=dev)
f, s = svd_truncated_device(sb.DeviceTensor(x.data, (m, p, n)), ranks, k * n, keep_values=True)
s = s.cpu().numpy().reshape((min(m, p), n), order="F")
ud = f.u_data.cpu().numpy()
gd = f.g_data.cpu().numpy()
uo = f.u_off.cpu().numpy()
go = f.g_off.cpu().numpy()
nbad = 0
for i in range(n):
    ai = ahat[:, :, i]
    sl = np.linalg.svd(ai, compute_uv=False)
    u = ud[uo[i]:uo[i] + m * k].reshape((m, k), order="F")
    g = gd[go[i]:go[i] + k * p].reshape((k, p), order="F")
    err2 = np.sum((ai - u @ g) ** 2)
    tail = np.sum(sl[k:] ** 2)
    orth = np.abs(u.T @ u - np.diag(np.sum(u * u, axis=0))).max()
    bad = abs(err2 - tail) > 1e-10 * max(tail, 1e-300) + 1e-20
    if bad or i < 2:
      print(f"{'BAD ' if bad else ''}slice {i}: err2 {err2:.6e} tail {tail:.6e} rel {(err2 - tail) / max(tail, 1e-300):.3e} "
            f"sig[k-2:k+2] {sl[k-2:k+2]} ours {s[k-2:k+2, i]} |dsig|max {np.abs(s[:k+4, i]-sl[:k+4]).max():.2e} "
            f"uorth {orth:.1e}")
    if bad and nbad < 3:
      nbad += 1
      uu, sl2, vt = np.linalg.svd(ai)
      sv = s[:k, i]
      vv = (g / np.where(sv > 0, sv, 1.0)[:, None]).T   # p x k
      print("   sigma[:k]", np.array2string(sl[:k], precision=6, max_line_width=400))
      # residual ||A v_j - sigma_j u_j|| / sigma_j and ||A^T A v_j - s^2 v_j|| per column
      res = [np.linalg.norm(ai.T @ (ai @ vv[:, j]) - sv[j] ** 2 * vv[:, j]) / sv[j] ** 2 for j in range(k)]
      print("   vres", np.array2string(np.array(res), precision=1, max_line_width=400))
      print("   vnorm", np.array2string(np.linalg.norm(vv, axis=0), precision=3, max_line_width=400))
