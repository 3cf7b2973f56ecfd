"""Sturm sweeps per warp of the sigma kernel on the c2 step's kept slices:
phase A (multisection), B (Laguerre), C (bisection to the end)."""
import json, sys
import torch
sys.path.insert(0, ".")
import paper_2605_16058_b200 as sb
from paper_2605_16058_b200 import _native as nat, compress as cp
from paper_2605_16058_b200.configs import config2
from paper_2605_16058_b200.mode_product import forward_device
from paper_2605_16058_b200.slice_svd import svd_values_device
a = config2(nlat=361, nlon=720, nt=1024, seed=0)
ts = sb.TransformSet.build(a.shape, "dct")
x = sb.DeviceTensor.from_host(sb.DenseTensor(a, copy=False), torch.device("cuda", 0))
ah = forward_device(x, ts)
m, p, n = a.shape
sel = cp.prune_select(sb.DeviceTensor(ah.data, a.shape), 1e-2)
kid = torch.from_numpy(sel[0]).to(ah.device)
sub = sb.DeviceTensor(ah.data.view(n, m * p).index_select(0, kid).reshape(-1), (m, p, int(kid.numel())))
lib = nat.load()
lib.starm_svd_tune(-1, -1, -1, 1)
svd_values_device(sub); torch.cuda.synchronize(); nat.svd_stats(reset=True)
svd_values_device(sub); torch.cuda.synchronize()
st = nat.svd_stats(reset=True)
warps = int(kid.numel()) * ((361 + 31) // 32)
print("slices", int(kid.numel()), "warps", warps, "mean sweeps per warp: A", st["sweeps"] / warps, "B", st["pairs"] / warps, "C", st["rotated"] / warps, "max-coded", st["cyc_final"])
