"""Experiment: c2 reduce kernel (tune mode 3) with fewer CTAs in flight
(STARM_REDUCE_SLOTS) -- does an L2-resident working set shorten each slice?
Prints ms per launch and per-slice QR / band cycles from the kernel counters."""
import os
import subprocess
import sys

if len(sys.argv) > 1:
    import torch
    sys.path.insert(0, ".")
    import paper_2605_16058_b200 as sb
    from paper_2605_16058_b200 import _native as nat
    from paper_2605_16058_b200.configs import config2
    from paper_2605_16058_b200.mode_product import forward_device
    from paper_2605_16058_b200.slice_svd import svd_values_device
    a = config2(nlat=361, nlon=720, nt=1024, seed=0)
    ts = sb.TransformSet.build(a.shape, "dct")
    x = sb.DeviceTensor.from_host(sb.DenseTensor(a, copy=False), torch.device("cuda", 0))
    ah = sb.DeviceTensor(forward_device(x, ts).data, a.shape)
    lib = nat.load()
    lib.starm_svd_tune(-1, -1, 3, -1)
    svd_values_device(ah)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    svd_values_device(ah)
    e1.record()
    e1.synchronize()
    ms = e0.elapsed_time(e1)
    lib.starm_svd_tune(-1, -1, -1, 1)
    nat.svd_stats(reset=True)
    svd_values_device(ah)
    st = nat.svd_stats(reset=True)
    n = max(st["slices"], 1) if st["slices"] else 1024
    print(f"slots {os.environ.get('STARM_REDUCE_SLOTS', 'all')}: {ms:.2f} ms; per slice Mcycles "
          f"load {st['cyc_load'] / 1024 / 1e6:.2f} qr {st['cyc_qr'] / 1024 / 1e6:.2f} "
          f"band {st['cyc_band'] / 1024 / 1e6:.2f} pfact {st['cyc_pfact'] / 1024 / 1e6:.2f} "
          f"trail {st['cyc_trail'] / 1024 / 1e6:.2f} right {st['cyc_right'] / 1024 / 1e6:.2f}",
          flush=True)
else:
    for slots in ["148", "120", "96", "74", "48"]:
        subprocess.run([sys.executable, __file__, "run"], env=dict(os.environ, STARM_REDUCE_SLOTS=slots))
