"""One warm + one measured step of a BASELINE workload (device-resident
input) -- target for ncu launch lists.  usage: run_wl_step.py c1|c2|c3|c4|c5"""
import sys

import torch

sys.path.insert(0, ".")
from paper_2605_16058_b200.workloads import make_workload

wl = make_workload(sys.argv[1] if len(sys.argv) > 1 else "c2")
x = wl.device_input(torch.device("cuda", 0))
wl.extra.pop("ahat", None)
for _ in range(2):
    r = wl.step(x)
torch.cuda.synchronize()
print("ok", wl.name, r.factors.total_rank)
