"""Which host call of a tsvdm_tolerance step occasionally stalls?  Wraps the
step's host-side entry points with wall-clock timers for 40 steps and prints
the max / median per function."""
import collections, functools, json, statistics, sys, time

import torch

sys.path.insert(0, ".")
import paper_2605_16058_b200 as sb
from paper_2605_16058_b200 import compress
from paper_2605_16058_b200.configs import config2

times = collections.defaultdict(list)


def wrap(mod, name, label=None):
    f = getattr(mod, name)

    @functools.wraps(f)
    def g(*a, **k):
        t0 = time.perf_counter()
        try:
            return f(*a, **k)
        finally:
            times[label or name].append(1e3 * (time.perf_counter() - t0))
    setattr(mod, name, g)


for nm in ("forward_device", "svd_values_device", "threshold_device", "_summary", "svd_truncated_device",
           "_finish", "_state_fits", "check_status"):
    if hasattr(compress, nm):
        wrap(compress, nm)
wrap(torch.cuda, "mem_get_info", "mem_get_info")
a = config2(nlat=361, nlon=720, nt=1024, seed=0)
ts = sb.TransformSet.build(a.shape, "dct")
x = sb.DeviceTensor.from_host(sb.DenseTensor(a, copy=False), torch.device("cuda", 0))
for _ in range(3):
    sb.tsvdm_tolerance(x, ts, 1e-2)
torch.cuda.synchronize()
times.clear()
step = []
for k in range(40):
    t0 = time.perf_counter()
    sb.tsvdm_tolerance(x, ts, 1e-2)
    torch.cuda.synchronize()
    step.append(1e3 * (time.perf_counter() - t0))
out = {k: {"max": round(max(v), 2), "med": round(statistics.median(v), 2), "n": len(v)} for k, v in times.items()}
out["step"] = {"max": round(max(step), 2), "med": round(statistics.median(step), 2)}
print(json.dumps(out))
