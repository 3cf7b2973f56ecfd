"""c3 (1024x1024x512, Haar M, rank 32): per-step time with CUDA events
(2 warm-up, 3 timed) -- quick A/B target (e.g. STARM_BULGE_CLUSTER=0)."""
import sys
import torch
sys.path.insert(0, ".")
import paper_2605_16058_b200 as sb
from paper_2605_16058_b200 import configs
from paper_2605_16058_b200.transform_set import validate_transform

a, mm = configs.config3()
ts = sb.TransformSet((validate_transform(mm),))
x = sb.DeviceTensor.from_host(sb.DenseTensor(a, copy=False), torch.device("cuda", 0))
for _ in range(2):
    c = sb.tsvdm_fixed_rank(x, ts, 32)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(3):
    c = sb.tsvdm_fixed_rank(x, ts, 32)
e1.record(); e1.synchronize()
print("c3 step ms", e0.elapsed_time(e1) / 3, "total rank", c.factors.total_rank, "rel err", c.relative_error())
