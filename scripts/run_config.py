"""Full-size run of one BASELINE config on cuda:0 through the public API:
time the compression (device-resident input) and check the realised error
against the energy identity  relerr^2 = discarded / total  (orthogonal M).

usage: python scripts/run_config.py c1|c2|c3|c4|c5 [reps] [tol]
"""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2605_16058_b200 as sb
from paper_2605_16058_b200 import configs
from paper_2605_16058_b200.compress import reconstruct_device, relative_error_device
from paper_2605_16058_b200.transform_set import validate_transform

name = sys.argv[1]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
dev = torch.device("cuda", 0)
t0 = time.time()
if name == "c1":
    a = configs.config1()
    ts = sb.TransformSet.build(a.shape, "dct")
    run = lambda x: sb.tsvdm_fixed_rank(x, ts, 10)
elif name == "c2":
    a = configs.config2()
    ts = sb.TransformSet.build(a.shape, "dct")
    run = lambda x: sb.tsvdm_tolerance(x, ts, 1e-2)
elif name == "c3":
    a, mm = configs.config3()
    ts = sb.TransformSet((validate_transform(mm),))
    run = lambda x: sb.tsvdm_fixed_rank(x, ts, 32)
elif name == "c5":
    ahat, mm = configs.config5_transform_domain()
    ts = sb.TransformSet((validate_transform(mm),))
    # original-domain tensor = ahat x_3 M^T, formed on the device
    xh = sb.DeviceTensor.from_host(sb.DenseTensor(ahat, copy=False), dev)
    del ahat
    from paper_2605_16058_b200.mode_product import inverse_device
    a = None
    xdev = inverse_device(xh, ts)
    del xh
    run = lambda x: sb.tsvdm_fixed_rank(x, ts, 16)
    if len(sys.argv) > 3 and sys.argv[3] == "tol":
        run = lambda x: sb.tsvdm_tolerance(x, ts, 1e-4)
elif name == "c4":
    # SURVEY 8c "Config 4 restatement": float32 input upcast to float64 (tensor.py:87), the
    # non-orthonormal M applied as a raw-matrix ttm, values -> threshold -> truncated factors,
    # reconstruction with the explicit M^-1 (not M^T)
    a32, mm, minv = configs.config4()
    a = np.asfortranarray(a32, dtype=np.float64)  # upcast like the reference (tensor.py:87)
    del a32
    eps4 = 1e-3

    from paper_2605_16058_b200.compress import _summary, threshold_device
    from paper_2605_16058_b200.slice_svd import svd_truncated_device, svd_values_device

    def run(x):
        # tsvdm_tolerance's memory-efficient schedule (values pass keeping each
        # slice's factorisation state -> device threshold -> truncated pass from
        # the state) with the raw M, which a TransformSet would reject
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
        ev[0].record()
        ahat = sb.ttm(x, 2, mm)
        ev[1].record()
        s, state = svd_values_device(ahat, keep_state=True)
        ev[2].record()
        m_, p_, n_ = ahat.dims
        ranks, scal, j, _, _ = threshold_device(s, min(m_, p_), n_, eps4)
        tau, disc, tot, total_rank = _summary(ranks, scal)
        thr = sb.ThresholdResult(None, None, int(j.item()), tau, ranks, disc, tot)
        ev[3].record()
        f, _ = svd_truncated_device(ahat, ranks, total_rank, state=state)
        del state
        ev[4].record()
        ev[4].synchronize()
        print("    stages ms: " + ", ".join(f"{k} {ev[i].elapsed_time(ev[i + 1]):.1f}" for i, k in
                                          enumerate(("ttm", "values", "threshold", "truncated"))))
        return ahat, thr, f
else:
    raise SystemExit(f"unknown config {name}")
if a is not None:
    xdev = sb.DeviceTensor.from_host(sb.DenseTensor(a, copy=False), dev)
    del a
print(f"{name}: dims {xdev.dims}, setup {time.time() - t0:.1f}s", flush=True)
for i in range(reps):
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    c = run(xdev)
    e1.record()
    e1.synchronize()
    ms = e0.elapsed_time(e1)
    tr = c[2].total_rank if name == "c4" else c.factors.total_rank
    print(f"  rep {i}: {ms:.1f} ms  total_rank {tr}", flush=True)
if name == "c4":
    from paper_2605_16058_b200 import _native as nat
    ahat, thr, f = c
    m_, p_, n_ = xdev.dims
    chat = sb.DeviceTensor.empty(xdev.dims, dev)
    nat.call("starm_unpack_facewise_f64", f.u_data.data_ptr(), f.g_data.data_ptr(),
             f.ranks_dev.data_ptr(), f.u_off.data_ptr(), f.g_off.data_ptr(), m_, p_, n_,
             chat.data.data_ptr(), nat.stream_ptr(dev))
    err_t = relative_error_device(ahat, chat)
    rec = sb.ttm(chat, 2, minv)
    err_o = relative_error_device(xdev, rec)
    pred = float(np.sqrt(thr.discarded_energy / thr.total_energy))
    print(f"  J {thr.j}  tau {thr.tau:.6g}  sum rank {f.total_rank} of {m_ * n_}")
    print(f"  transform-domain relerr {err_t:.10g}  predicted {pred:.10g}  diff {abs(err_t - pred):.3g}")
    print(f"  original-domain relerr {err_o:.10g} (M non-orthonormal: not bounded by eps)")
    ok = abs(err_t - pred) <= 1e-8 + 1e-6 * pred and err_t <= eps4
    print("OK" if ok else "MISMATCH")
    sys.exit(0 if ok else 1)
rec = reconstruct_device(c, dev)
err = relative_error_device(xdev, rec)
pred = float(np.sqrt(c.discarded_energy / c.total_energy))
print(f"  realised relerr {err:.10g}  predicted {pred:.10g}  diff {abs(err - pred):.3g}")
ok = abs(err - pred) <= 1e-8 + 1e-6 * pred
print("OK" if ok else "MISMATCH")
sys.exit(0 if ok else 1)
