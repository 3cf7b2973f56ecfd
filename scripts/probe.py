"""Quick device probe: FP64 DGEMM peak (cuBLAS reference point), K1 TTM on the
c2 geometry, K3 Jacobi SVD on c2-shaped slices."""
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2605_16058_b200 as sb
from paper_2605_16058_b200 import _native as nat


def evt_time(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    b.synchronize()
    return a.elapsed_time(b) / 1e3 / reps


out = {}
dev = torch.device("cuda", 0)
n = 8192
A = torch.randn(n, n, dtype=torch.float64, device=dev)
B = torch.randn(n, n, dtype=torch.float64, device=dev)
t = evt_time(lambda: torch.matmul(A, B), 3)
out["cublas_dgemm_tflops_burst"] = 2 * n**3 / t / 1e12
# sustained ~4 s
t0 = time.time(); k = 0
torch.cuda.synchronize()
a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
a.record()
while time.time() - t0 < 4.0:
    torch.matmul(A, B); k += 1
b.record(); b.synchronize()
out["cublas_dgemm_tflops_sustained"] = 2 * n**3 * k / (a.elapsed_time(b) / 1e3) / 1e12
del A, B

# K1 on the c2 geometry
rows, inner = 361 * 720, 1024
src = torch.randn(rows * inner, dtype=torch.float64, device=dev)
mat = torch.randn(inner, inner, dtype=torch.float64, device=dev)
dst = torch.empty_like(src)
st = nat.stream_ptr(dev)
f = lambda: nat.call("starm_ttm_f64", src.data_ptr(), mat.data_ptr(), dst.data_ptr(), rows, inner, 1, inner, st)
t = evt_time(f, 5)
out["ttm_c2_ms"] = t * 1e3
out["ttm_c2_tflops"] = 2 * inner * inner * rows / t / 1e12
# check vs cuBLAS
ref = (mat @ src.view(inner, rows))
out["ttm_c2_relerr_vs_cublas"] = float((dst.view(inner, rows) - ref).norm() / ref.norm())
t = evt_time(lambda: torch.matmul(mat, src.view(inner, rows)), 3)
out["cublas_ttm_c2_tflops"] = 2 * inner * inner * rows / t / 1e12
del src, dst, ref

# K3 values on c2-shaped random slices
for (m, p, N) in [(361, 720, 148), (256, 256, 64), (8192, 64, 148)]:
    x = sb.DeviceTensor(torch.randn(m * p * N, dtype=torch.float64, device=dev), (m, p, N))
    from paper_2605_16058_b200.slice_svd import svd_values_device
    t = evt_time(lambda: svd_values_device(x), 1)
    out[f"svd_values_{m}x{p}x{N}_ms"] = t * 1e3
print(json.dumps(out, indent=1))
