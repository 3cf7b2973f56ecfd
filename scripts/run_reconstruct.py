"""c2: one compression, then the fused reconstruction + error twice (target
for ncu launch lists of starm_reconstruct_f64)."""
import sys, time
import torch
sys.path.insert(0, ".")
import paper_2605_16058_b200 as sb
from paper_2605_16058_b200.configs import config2

a = config2(nlat=361, nlon=720, nt=1024, seed=0)
ts = sb.TransformSet.build(a.shape, "dct")
x = sb.DeviceTensor.from_host(sb.DenseTensor(a, copy=False), torch.device("cuda", 0))
c = sb.tsvdm_tolerance(x, ts, 1e-2)
for _ in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    rec, err = sb.reconstruct_fused(c, a=x)
    torch.cuda.synchronize(); print("reconstruct_fused ms", (time.perf_counter() - t0) * 1e3, err)
