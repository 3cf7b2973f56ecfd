"""Step-time spikes: are they host-side or GPU-side?  Times 40 full steps,
then 40 launches of the values pass alone (device-only, no host syncs inside
a launch sequence) with per-iteration CUDA events, and samples NVML clocks /
event reasons every 20 ms meanwhile."""
import json, sys, threading, time

import torch

sys.path.insert(0, ".")
import paper_2605_16058_b200 as sb
from paper_2605_16058_b200.configs import config2
from paper_2605_16058_b200.mode_product import forward_device
from paper_2605_16058_b200.slice_svd import svd_values_device

import pynvml
pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(0)
samples = []
stop = threading.Event()


def sampler():
    while not stop.is_set():
        t = time.perf_counter()
        samples.append((t, pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM),
                        pynvml.nvmlDeviceGetCurrentClocksEventReasons(h),
                        pynvml.nvmlDeviceGetPowerUsage(h)))
        stop.wait(0.02)


a = config2(nlat=361, nlon=720, nt=1024, seed=0)
ts = sb.TransformSet.build(a.shape, "dct")
x = sb.DeviceTensor.from_host(sb.DenseTensor(a, copy=False), torch.device("cuda", 0))
for _ in range(3):
    sb.tsvdm_tolerance(x, ts, 1e-2)
torch.cuda.synchronize()
th = threading.Thread(target=sampler, daemon=True)
th.start()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(41)]
hs = []
ev[0].record()
for k in range(40):
    hs.append(time.perf_counter())
    sb.tsvdm_tolerance(x, ts, 1e-2)
    ev[k + 1].record()
torch.cuda.synchronize()
steps = [round(ev[k].elapsed_time(ev[k + 1]), 2) for k in range(40)]
ahat = sb.DeviceTensor(forward_device(x, ts).data, a.shape)
svd_values_device(ahat)
torch.cuda.synchronize()
ev[0].record()
for k in range(40):
    svd_values_device(ahat)
    ev[k + 1].record()
torch.cuda.synchronize()
vals = [round(ev[k].elapsed_time(ev[k + 1]), 2) for k in range(40)]
stop.set()
th.join()
clk = sorted(set(s[1] for s in samples))
reasons = sorted(set(s[2] for s in samples))
print(json.dumps({"steps": steps, "values_pass": vals, "sm_clocks_seen": clk, "reason_bits_seen": reasons,
                  "power_mw_max": max(s[3] for s in samples), "n_samples": len(samples)}))
