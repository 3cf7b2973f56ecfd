#!/usr/bin/env python
"""Benchmark: t-SVDM compression throughput (input GB/s) on B200.

Workloads (``--config``, paper_2605_16058_b200/workloads.py; BASELINE.json
configs): c1 fixed rank 10 (256x256x64), c2 tolerance 1e-2 (361x720x1024,
DCT: the default -- BASELINE's metric is quoted on configs[1]), c3 fixed
rank 32 (1024^2 x 512, Haar), c4 tolerance 1e-3 (512^2 x 2048 X-ray-like,
raw invertible M), c5 fixed rank 16 / c5t tolerance 1e-4 (8192x64x4096,
Haar).  Seeded synthetic data of each config's shape and distribution.

One step = one compression call (forward transform -> slice SVDs ->
threshold -> packed factors).
  value : input bytes / s with the tensor already resident in HBM (every
          config's input exceeds the 126 MB L2 except c1, 33.5 MB: c1 steps
          are separated by an L2 flush, a 256 MB write, outside the events)
  e2e   : the same through the drop-in host call (DenseTensor in from pinned
          memory, host CompressedTensor out): H2D of the input and D2H of the
          packed factors inside every timed step.  ``e2e_stream`` is the
          pipelined host API (tsvdm_tolerance_stream: H2D of step k+1 under
          step k), tolerance configs only.

Multi-GPU.  ``--gpus N`` (N > 1) without a torchrun environment relaunches
itself under ``torch.distributed.run`` with N local ranks.  Under torchrun
the default is north_star's split of ONE tensor (sharded.py): fibre-local
transform, NCCL all-to-all to slice ownership, per-rank SVDs, all-gathered
sigma, replicated threshold/energies ("scaling": "strong");
``--replicas`` runs N independent tensors instead ("weak").  Time = max
over ranks of the device-timed region.

``--impl reference`` times the reference algorithm on the host cores: the
oracle port (oracle/, numpy + LAPACK dgesvd exactly like the reference
package; the reference itself is not present on the GPU box) on a bounded
per-slice sample of the same workload, rank 0 only.
"""

from __future__ import annotations

import argparse
import gc
import json
import math
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

UNIT = "GB/s"


def metric_name(cfg):
    return f"t-SVD input GB/s ({cfg} t-SVDM, device-resident input)"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c2", choices=["c1", "c2", "c3", "c4", "c5", "c5t"])
    ap.add_argument("--cpu-sample-slices", type=int, default=0,
                    help="slices in the CPU sample (0 = auto, ~10-20 s of CPU work)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--replicas", action="store_true",
                    help="N>1: N independent tensors (weak scaling) instead of one sharded tensor")
    ap.add_argument("--sharded", action="store_true",
                    help="run the sharded pipeline even at N=1 (world size 1 over NCCL)")
    ap.add_argument("--dry-run", action="store_true",
                    help="launch plumbing only (gloo on CPU): ranks join, plan checked, no compute")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def relaunch_under_torchrun(args):
    """``--gpus N`` from a plain ``python bench.py``: re-exec under
    torch.distributed.run with N local ranks (127.0.0.1 rendezvous)."""
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1", f"--master-port={port}",
           os.path.abspath(__file__)] + sys.argv[1:]
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    env.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
    return subprocess.call(cmd, env=env)


# ------------------------------------------------------------ CPU baseline

def cpu_sample(wl, nslices, threads, a=None):
    """The reference algorithm (oracle restatement, numpy + LAPACK dgesvd)
    on a per-slice sample of workload ``wl``: the forward transform
    restricted to the first ``nslices`` OUTPUT slices (M[:S] @ A_(3), full
    inner dimension, all BLAS threads), then per slice the SVD the reference
    runs (values pass + truncated pass for tolerance; truncated with
    keep_values for fixed rank; 1 core: scipy's dgesvd wrapper holds the
    GIL) and the threshold over the sample.  Returns (seconds, bytes of
    input represented)."""
    import oracle
    from threadpoolctl import threadpool_limits
    m, p, n = wl.dims
    if a is None:
        a = wl.host
    if wl.transform == "dct":
        mat = oracle.dct_matrix(n)
    elif wl.transform == "raw":
        mat = wl.mat
    else:
        mat = wl.ts[0].matrix
    mat = np.ascontiguousarray(mat[:nslices, :])
    t0 = time.perf_counter()
    with threadpool_limits(limits=threads, user_api="blas"):
        flat = a.reshape(-1, order="F").reshape(n, m * p)
        ahat = (mat @ flat).reshape(-1).reshape((m, p, nslices), order="F")
    with threadpool_limits(limits=1, user_api="blas"):
        if wl.kind == "tolerance":
            oracle.tsvdm_tolerance(None, None, float(wl.param), ahat=ahat)
        else:
            ranks = np.full(nslices, int(wl.param), dtype=np.int64)
            oracle.svd_truncated_slices(ahat, ranks, keep_values=True)
    dt = time.perf_counter() - t0
    return dt, nslices * m * p * (wl.in_bytes // (m * p * n))


def cpu_info():
    model = ""
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return model, os.cpu_count() or 1


def per_slice_cpu_seconds(wl):
    """Rough 1-core dgesvd seconds per slice, used only to
    size the sample to ~10-20 s."""
    m, p, _ = wl.dims
    return max(1e-3, 0.27 * (m * p * min(m, p)) / (361 * 720 * 361))


def host_for_cpu(wl):
    """Host input for the CPU sample (c5 is formed on the device: only the
    first few hundred time steps' worth of host data exist otherwise)."""
    if wl.host is not None:
        return wl.host
    import oracle
    ahat = wl.extra["ahat"]
    return oracle.ttm(ahat, 2, wl.extra["mat"].T)


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    from paper_2605_16058_b200.workloads import make_workload
    wl = make_workload(args.config, seed=0)
    a = host_for_cpu(wl)
    model, cores = cpu_info()
    budget = 150.0 / max(args.steps + args.warmup, 1)
    s = args.cpu_sample_slices or max(2, int(budget / per_slice_cpu_seconds(wl)))
    s = min(s, wl.dims[2])
    for _ in range(args.warmup):
        cpu_sample(wl, max(1, s // 4), cores, a)
    times, nbytes = [], 0
    for _ in range(args.steps):
        dt, nbytes = cpu_sample(wl, s, cores, a)
        times.append(dt)
    v = nbytes / statistics.mean(times) / 1e9
    line = {
        "impl": "reference", "metric": metric_name(args.config), "value": v, "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * statistics.mean(times), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": f"synthetic (workloads.{args.config}, seed 0)",
        "config": {"workload": wl.describe, "global_batch": 1, "seq_len": wl.dims[2],
                   "parallelism": "cpu"},
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "port",
                         "sample": f"first {s} of {wl.dims[2]} transform-domain slices per step: "
                                   f"restricted transform (all {cores} BLAS threads) + dgesvd "
                                   f"passes (1 core: the reference's f2py wrapper holds the GIL) "
                                   f"+ threshold; CPU {model}"},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    emit(line)


# ------------------------------------------------------------ GPU arm helpers

class ClockSampler:
    """SM clocks and clock-event (throttle) reasons sampled every 200 ms during
    the timed region through NVML in a background thread (nvidia-smi's own
    start-up takes driver locks that stall the stream being timed; NVML is
    initialised and queried once before the region starts).  Falls back to
    an ``nvidia-smi -lms 200`` subprocess when pynvml is missing."""

    REASONS = (("hw_slowdown", 0x8), ("hw_thermal_slowdown", 0x40),
               ("sw_thermal_slowdown", 0x20), ("sw_power_cap", 0x4))
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index, pci_bus_id=None):
        self.index = index
        self.pci = pci_bus_id
        self.samples = []  # (sm_mhz, max_mhz, reason bits)
        self.lines = []
        self.proc = None
        self._stop = threading.Event()
        self._thread = None

    def _nvml_handle(self):
        import pynvml
        pynvml.nvmlInit()
        if self.pci:
            try:
                return pynvml, pynvml.nvmlDeviceGetHandleByPciBusId(self.pci)
            except pynvml.NVMLError:
                pass
        return pynvml, pynvml.nvmlDeviceGetHandleByIndex(self.index)

    def __enter__(self):
        if os.environ.get("STARM_BENCH_NO_SMI"):
            return self
        try:
            nv, h = self._nvml_handle()
        except Exception:
            return self._enter_smi()
        mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
        reasons = getattr(nv, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
            nv.nvmlDeviceGetCurrentClocksThrottleReasons

        def query():
            return nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM), mx, reasons(h)

        query()  # warm the NVML path before the region starts
        self.query_ms = []

        def run():
            while not self._stop.is_set():
                t0 = time.perf_counter()
                try:
                    self.samples.append(query())
                except Exception:
                    pass
                self.query_ms.append(round(1e3 * (time.perf_counter() - t0), 3))
                self._stop.wait(0.2)

        self._thread = threading.Thread(target=run, daemon=True)
        self._thread.start()
        return self

    def _enter_smi(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except (OSError, ValueError):
            self.proc = None
            return self
        first = threading.Event()

        def pump():
            for line in self.proc.stdout:
                if line.strip():
                    self.lines.append(line)
                    first.set()
            first.set()

        self._thread = threading.Thread(target=pump, daemon=True)
        self._thread.start()
        first.wait(timeout=10)
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
        if self._thread is not None:
            self._thread.join(timeout=5)

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        for s_mhz, m_mhz, bits in self.samples:
            sm.append(float(s_mhz))
            mx = max(mx, float(m_mhz))
            for nm, bit in self.REASONS:
                if bits & bit:
                    reasons.add(nm)
        names = [nm for nm, _ in self.REASONS]
        for line in self.lines:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx = max(mx, float(parts[1]))
            except ValueError:
                continue
            for nm, val in zip(names, parts[3:7]):
                if val.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm),
                "source": "nvml" if self.samples else ("nvidia-smi" if self.lines else None)}


def pci_bus_id(torch, dev):
    try:
        p = torch.cuda.get_device_properties(dev)
        return "%08X:%02X:%02X.0" % (p.pci_domain_id, p.pci_bus_id, p.pci_device_id)
    except Exception:
        return None


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs"
    except (OSError, KeyError, ValueError):
        return 7700.0, "B200_PROFILING.md fallback"


def profiled_traffic(kernel, cfg):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of ``kernel``
    on this workload, from the committed ncu --set full capture summary."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            d = json.load(f)
        return d.get(f"{cfg}/{kernel}", d.get(kernel) if cfg == "c2" else None)
    except (OSError, ValueError):
        return None


def wave_text(slices, sms):
    """How the reduce launch maps slices to SMs (svd_f64.cu: one CTA per slice,
    or a cluster of 2 / 4 / 8 CTAs per slice when slices <= SMs / 2; a last
    partial wave of a multi-wave launch also runs on clusters)."""
    if slices <= sms // 2:
        c = 1
        while c < 8 and slices * 2 * c <= sms:
            c *= 2
        return f"{slices} slices on {sms} SMs ({c}-CTA cluster per slice)"
    waves = -(-slices // sms)
    return f"{slices} slices on {sms} SMs (one CTA per slice, {waves} wave{'s' if waves > 1 else ''})"


def fp64_peak(torch, dev):
    """cuBLAS DGEMM rate on this box (the FP64 denominator; MEASURED_PEAKS.json
    has no FP64 entry)."""
    n = 4096
    a = torch.randn(n, n, dtype=torch.float64, device=dev)
    b = torch.randn(n, n, dtype=torch.float64, device=dev)
    for _ in range(2):
        torch.matmul(a, b)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    k = 10
    for _ in range(k):
        torch.matmul(a, b)
    e1.record()
    e1.synchronize()
    return 2 * n ** 3 * k / (e0.elapsed_time(e1) / 1e3) / 1e12


def timed(torch, fn, reps=1):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        out = fn()
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) / 1e3 / reps, out


def host_available_bytes():
    try:
        import psutil
        return psutil.virtual_memory().available
    except Exception:
        return 0


# ------------------------------------------------------------ GPU arm (1 tensor / rank)

def run_ours(args):
    import torch
    import torch.distributed as dist

    rank, world, local = dist_env()
    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl")
    dev = torch.device("cuda", local if world > 1 else 0)
    torch.cuda.set_device(dev)

    import paper_2605_16058_b200 as sb
    from paper_2605_16058_b200 import _native as nat
    from paper_2605_16058_b200.workloads import make_workload
    from paper_2605_16058_b200.slice_svd import svd_values_device

    wl = make_workload(args.config, seed=rank)
    x = wl.device_input(dev)
    wl.extra.pop("ahat", None)
    m, p, n = wl.dims
    in_bytes = wl.in_bytes
    is_tol = wl.kind == "tolerance"
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev) if in_bytes < (256 << 20) else None
    torch.cuda.synchronize()

    for _ in range(max(args.warmup, 1)):
        res = wl.step(x)
    torch.cuda.synchronize()
    lib = nat.load()
    lib.starm_launch_count_reset()

    # ---- device-resident timed region
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    gc.collect()
    gc.disable()  # no collector pauses inside the timed host loop
    with ClockSampler(dev.index, pci_bus_id(torch, dev)) as clk:
        for k in range(args.steps):
            if flush is not None:
                flush.fill_(k & 0xFF)   # L2 flush between steps (outside the events)
            starts[k].record()
            res = wl.step(x)
            ends[k].record()
        ends[-1].synchronize()
    torch.cuda.synchronize()
    gc.enable()
    step_ms = [round(starts[k].elapsed_time(ends[k]), 3) for k in range(args.steps)]
    launches = lib.starm_launch_count_reset() // max(args.steps, 1)
    t_dev = sum(step_ms) / 1e3
    if world > 1:
        tt = torch.tensor([t_dev], device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_dev = float(tt.item())
        dist.barrier()
    value = world * args.steps * in_bytes / t_dev / 1e9
    total_rank = res.factors.total_rank
    # validity of the timed result (outside the timed region): the realised
    # error equals the energy bookkeeping and meets the tolerance
    realised, recorded = wl.realised_error(x, res)
    if not abs(realised - recorded) <= 1e-8 * max(1.0, recorded) or (is_tol and not realised <= wl.param):
        raise SystemExit(f"bench: invalid result: realised error {realised} vs recorded {recorded}")

    # ---- reconstruction + error, timed separately
    t_rec, _ = timed(torch, lambda: wl.realised_error(x, res), reps=2)

    # ---- stage split and the dominant kernel
    stages = {}
    if is_tol and wl.transform != "raw":
        clock = sb.StageClock()
        wl.step(x, clock=clock)
        stages = {k: round(v * 1e3, 3) for k, v in clock.seconds.items()}
    t_fwd, ahat = timed(torch, lambda: wl.forward(x))
    ahat3 = sb.DeviceTensor(ahat.data, (m, p, n))
    # tolerance steps run the values pass on the slices the certified pruning
    # keeps (compress.prune_select): time the kernels on that same subset
    n_svd = n
    if is_tol and wl.transform != "raw":
        from paper_2605_16058_b200 import compress
        sel = compress.prune_select(ahat3, float(wl.param)) if compress.PRUNE else None
        if sel is not None:
            kid = torch.from_numpy(sel[0].astype(np.int64)).to(dev)
            n_svd = int(kid.numel())
            ahat3 = sb.DeviceTensor(ahat3.data.view(n, m * p).index_select(0, kid).reshape(-1),
                                    (m, p, n_svd))
    svd_values_device(ahat3)
    t_values, _ = timed(torch, lambda: svd_values_device(ahat3))
    # the reduce kernel alone (tune mode 3 stops the values pass after it);
    # tall-skinny slices (c5: 8192 x 64) take the TSQR route instead, whose
    # row-block QR + stacked reduce is not what mode 3 times: skipped there
    tsqr = ((max(m, p) + 63) // 64) * 64 > 1344 and min(m, p) <= 256
    t_red = None
    if not tsqr:
        lib.starm_svd_tune(-1, -1, 3, -1)
        try:
            svd_values_device(ahat3)
            t_red, _ = timed(torch, lambda: svd_values_device(ahat3), reps=2)
        finally:
            lib.starm_svd_tune(-1, -1, 1, -1)
    # ---- the same step and reduce launch WITHOUT the certified pruning (what
    # the reference's schedule does: every slice factored), for the record
    unpruned = None
    if n_svd < n:
        from paper_2605_16058_b200 import compress
        full3 = sb.DeviceTensor(ahat.data, (m, p, n))
        lib.starm_svd_tune(-1, -1, 3, -1)
        try:
            svd_values_device(full3)
            t_red_full, _ = timed(torch, lambda: svd_values_device(full3), reps=2)
        finally:
            lib.starm_svd_tune(-1, -1, 1, -1)
        del full3
        compress.PRUNE = False
        try:
            wl.step(x)
            t_full, _ = timed(torch, lambda: wl.step(x), reps=3)
        finally:
            compress.PRUNE = True
        unpruned = {"ms_per_step": t_full * 1e3, "value": in_bytes / t_full / 1e9, "unit": UNIT,
                    "reduce_ms": t_red_full * 1e3, "slices": n,
                    "what": "STARM_PRUNE=0: all slices through the values pass, as the "
                            "reference's schedule (tsvdm.py:268-321); same ranks and factors"}
    del ahat, ahat3
    f_ttm, f_svd, f_lapack = wl.flops(total_rank)
    a_, b_ = max(m, p), min(m, p)
    # Sigma-only GVL count = the reduce kernel's work, for the slices it factors
    # (all of them, or those the certified pruning keeps)
    f_red = n_svd * (2 * a_ * b_ ** 2 + 2 * b_ ** 3)
    f_svd_step = f_svd - (n - n_svd) * (2 * a_ * b_ ** 2 + 2 * b_ ** 3)
    peak = fp64_peak(torch, dev)
    hbm_peak, hbm_src = measured_peaks()
    dense = wl.transform != "dct"
    fwd_obj = {"ms": t_fwd * 1e3}
    if dense:
        fwd_obj.update(bound="tensor", kernel="gemm_f64_kernel (FP64 DMMA, 4-stage cp.async ring)",
                       achieved=f_ttm / t_fwd / 1e12, peak=peak, unit="TFLOP/s",
                       frac=f_ttm / t_fwd / 1e12 / peak, algorithmic_flops=f_ttm,
                       traffic=profiled_traffic("gemm_f64_kernel", args.config))
    else:
        dct_bytes = 2 * 8 * n * m * p
        fwd_obj.update(bound="hbm", kernel="dct1024_kernel + residual_gemm_kernel (tcgen05)",
                       achieved=dct_bytes / t_fwd / 1e9, peak=hbm_peak, unit="GB/s",
                       frac=dct_bytes / t_fwd / 1e9 / hbm_peak, algorithmic_bytes=dct_bytes,
                       traffic=profiled_traffic("dct1024_kernel", args.config))
    red_obj = None
    if t_red is not None:
        red_obj = {"bound": "tensor",
                   "kernel": "svd_reduce_kernel (Householder QR + band reduction, FP64 DMMA)",
                   "achieved": f_red / t_red / 1e12, "peak": peak, "unit": "TFLOP/s",
                   "frac": f_red / t_red / 1e12 / peak,
                   "traffic": profiled_traffic("svd_reduce_kernel", args.config),
                   "algorithmic_flops": f_red, "ms": t_red * 1e3, "slices": n_svd,
                   "wave": wave_text(n_svd, torch.cuda.get_device_properties(dev).multi_processor_count)}
    if unpruned is not None:
        f_full = n * (2 * a_ * b_ ** 2 + 2 * b_ ** 3)
        unpruned["reduce_achieved_tflops"] = f_full / (unpruned["reduce_ms"] / 1e3) / 1e12
        unpruned["reduce_frac"] = unpruned["reduce_achieved_tflops"] / peak
        unpruned["reduce_traffic"] = profiled_traffic("svd_reduce_kernel_unpruned", args.config)
    dominant = fwd_obj if (red_obj is None or (dense and t_fwd > t_red)) else red_obj
    roof = dict(dominant)
    roof["peak_source"] = ("cuBLAS DGEMM 4096^3 measured in this run (FP64 not in "
                           "MEASURED_PEAKS.json)") if roof["unit"] == "TFLOP/s" else hbm_src
    roof["forward_transform"] = fwd_obj
    roof["svd_reduce"] = red_obj
    roof["values_pass"] = {"ms": t_values * 1e3, "achieved": f_red / t_values / 1e12,
                           "kernels": "reduce + bulge chase + bisection/Laguerre"}
    bound_ms = 1e3 * (f_ttm / (peak * 1e12) if dense else 2 * 8 * n * m * p / (hbm_peak * 1e9)) \
        + 1e3 * f_svd_step / (peak * 1e12) + (1e3 * 8 * n * m * p / (hbm_peak * 1e9) if n_svd < n else 0.0)
    roof["step_bound_ms"] = bound_ms
    roof["step_frac"] = bound_ms / (1e3 * t_dev / args.steps * world / world)

    # ---- e2e through the drop-in host call: pinned host input -> H2D inside
    # the step -> host CompressedTensor (D2H of the packed factors)
    e2e = None
    e2e_stream = None
    if not args.no_e2e and host_available_bytes() > 3 * in_bytes:
        f32 = wl.host is not None and wl.host.dtype == np.float32
        pinned = torch.empty(m * p * n, dtype=torch.float32 if f32 else torch.float64,
                             pin_memory=True)
        if f32:
            pinned.numpy()[:] = wl.host.reshape(-1, order="F")
            host = pinned.numpy().reshape((m, p, n), order="F")   # float32 frames
        else:
            pinned.copy_(x.data, non_blocking=False)
            host = sb.DenseTensor(pinned.numpy().reshape((m, p, n), order="F"), copy=False)
        del x
        torch.cuda.empty_cache()

        def host_step():
            if wl.transform == "raw":
                xd = sb.DeviceTensor.from_host(host, dev)   # f32 H2D + device upcast
                r = wl.step(xd)
                return r.factors.to_host()
            if wl.kind == "fixed-rank":
                return sb.tsvdm_fixed_rank(host, wl.ts, int(wl.param)).factors
            return sb.tsvdm_tolerance(host, wl.ts, float(wl.param)).factors

        # two warm calls: results larger than 32 MB land in page-locked buffers
        # from torch's caching host allocator, and two results are alive at a
        # time (the previous one until the next is assigned)
        f = host_step()
        f = host_step()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            f = host_step()
        torch.cuda.synchronize()
        t_e2e = time.perf_counter() - t0
        d2h = int(f.u_data.nbytes + f.g_data.nbytes + f.ranks.nbytes)
        if world > 1:
            tt = torch.tensor([t_e2e], device=dev)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            t_e2e = float(tt.item())
        e2e = {"value": world * args.steps * in_bytes / t_e2e / 1e9, "unit": UNIT,
               "h2d_bytes_per_step": in_bytes, "d2h_bytes_per_step": d2h,
               "call": "tsvdm_tolerance / tsvdm_fixed_rank(DenseTensor) -> host CompressedTensor"}
        if is_tol and wl.transform != "raw":
            for _ in sb.tsvdm_tolerance_stream([host] * 2, wl.ts, float(wl.param)):
                pass
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            for _ in sb.tsvdm_tolerance_stream([host] * args.steps, wl.ts, float(wl.param)):
                pass
            torch.cuda.synchronize()
            t_s = time.perf_counter() - t0
            if world > 1:
                tt = torch.tensor([t_s], device=dev)
                dist.all_reduce(tt, op=dist.ReduceOp.MAX)
                t_s = float(tt.item())
            e2e_stream = {"value": world * args.steps * in_bytes / t_s / 1e9, "unit": UNIT,
                          "call": "tsvdm_tolerance_stream (H2D of step k+1 overlapped with step k)"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        model, cores = cpu_info()
        a_host = host_for_cpu(wl) if wl.host is not None else None
        if a_host is not None and a_host.dtype == np.float32:
            a_host = np.asfortranarray(a_host, dtype=np.float64)   # the reference upcasts
        if a_host is None and e2e is not None:
            a_host = host.array
        if a_host is not None:
            s = args.cpu_sample_slices or max(2, min(n, int(15.0 / per_slice_cpu_seconds(wl))))
            cpu_sample(wl, 1, cores, a_host)  # warm BLAS / LAPACK
            dt, nbytes = cpu_sample(wl, s, cores, a_host)
            cpu = {"value": nbytes / dt / 1e9, "unit": UNIT, "cores": cores, "kind": "port",
                   "sample": f"first {s} of {n} slices of {args.config}: restricted transform "
                             f"({cores} BLAS threads) + dgesvd passes (1 core, GIL) + threshold; "
                             f"{dt:.1f} s; CPU {model}"}

    if rank == 0:
        line = {
            "metric": metric_name(args.config), "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * t_dev / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "input_dtype": "f32" if wl.host is not None and wl.host.dtype == np.float32 else "f64",
            "data": f"synthetic (workloads.{args.config}, seed=rank)",
            "config": {"workload": wl.describe + ("; L2 flushed between steps" if flush is not None
                                                  else "; input > L2 (no flush needed)"),
                       "global_batch": world, "seq_len": n,
                       "parallelism": f"replicas x{world}" if world > 1 else "single"},
            "e2e": e2e, "e2e_stream": e2e_stream,
            "roofline": roof,
            "flops": {"transform": f_ttm, "svd_necessary": f_svd, "svd_lapack_equiv": f_lapack,
                      "svd_slices_factored": n_svd, "svd_in_step": f_svd_step,
                      "lapack_equiv_tflops": f_lapack / (t_dev / args.steps) / 1e12},
            "stages_ms": stages, "unpruned": unpruned,
            "reconstruct": {"ms": t_rec * 1e3, "what": "facewise U_i G_i + inverse transform + "
                                                       "K10 error sums (outside the timed region)"},
            "step_ms": step_ms, "clocks": clk.summary(), "gpu_launches": launches,
            "result": {"total_rank": total_rank, "relative_error": recorded,
                       "realised_error": realised,
                       **({"original_domain_error": wl.extra["orig_error"]}
                          if "orig_error" in wl.extra else {})},
            "cpu_baseline": cpu,
        }
        emit(line)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


# ------------------------------------------------------------ GPU arm (1 tensor sharded)

def sharded_block(cfg, plan):
    """This rank's (nf, N) fibre block of the workload's input (host), the
    transform, and (kind, param)."""
    import paper_2605_16058_b200 as sb
    from paper_2605_16058_b200 import configs as cf
    from paper_2605_16058_b200.sharded import scatter_fibres
    f0, f1 = plan.fibre_bounds()
    if cfg in ("c5", "c5t"):
        blk, mm = cf.config5_fibre_block(f0, f1, m=plan.m, p=plan.p, n=plan.n)
        tr = sb.validate_transform(mm)
        kind = ("fixed-rank", 16) if cfg == "c5" else ("tolerance", 1e-4)
        return blk, tr, kind, True     # block is in the M domain: A = Ahat x3 M^T on the device
    from paper_2605_16058_b200.workloads import make_workload
    wl = make_workload(cfg, seed=0)
    if wl.transform == "raw":
        raise SystemExit("bench: the sharded path needs an orthonormal transform (c4 is not)")
    blk = scatter_fibres(wl.host, plan)
    return blk, wl.ts[0], (wl.kind, wl.param), False


def run_sharded(args):
    """One tensor sharded over the ranks (paper_2605_16058_b200/sharded.py)."""
    import torch
    import torch.distributed as dist

    rank, world, local = dist_env()
    for k, v in (("MASTER_ADDR", "127.0.0.1"), ("MASTER_PORT", "29517"), ("RANK", "0"),
                 ("WORLD_SIZE", "1")):
        os.environ.setdefault(k, v)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    import paper_2605_16058_b200 as sb
    from paper_2605_16058_b200 import _native as nat
    from paper_2605_16058_b200.sharded import (DeviceOps, ShardPlan, reconstruct_sharded,
                                               relative_error_sharded, tsvdm_fixed_rank_sharded,
                                               tsvdm_tolerance_sharded)
    from paper_2605_16058_b200.workloads import make_workload
    dims = {"c1": (256, 256, 64), "c2": (361, 720, 1024), "c3": (1024, 1024, 512),
            "c5": (8192, 64, 4096), "c5t": (8192, 64, 4096)}[args.config]
    m, p, n = dims
    in_bytes = m * p * n * 8
    plan = ShardPlan(m, p, n, world, rank)
    blk, tr, (kind, param), m_domain = sharded_block(args.config, plan)
    ops = DeviceOps(tr, dev)
    x = torch.from_numpy(np.ascontiguousarray(blk.reshape(-1, order="F"))).to(dev)
    del blk
    if m_domain:
        x = ops.inverse(x, plan.nf, n).contiguous()    # A = Ahat x3 M^T, fibre-local
    torch.cuda.synchronize()

    def step(src):
        if kind == "fixed-rank":
            return tsvdm_fixed_rank_sharded(src, plan, ops, int(param), dist)
        return tsvdm_tolerance_sharded(src, plan, ops, float(param), dist)

    for _ in range(max(args.warmup, 1)):
        res = step(x)
    torch.cuda.synchronize()
    lib = nat.load()
    lib.starm_launch_count_reset()
    dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(dev.index, pci_bus_id(torch, dev)) as clk:
        e0.record()
        for _ in range(args.steps):
            res = step(x)
        e1.record()
        e1.synchronize()
    launches = lib.starm_launch_count_reset() // max(args.steps, 1)
    tt = torch.tensor([e0.elapsed_time(e1) / 1e3], device=dev)
    dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    t_dev = float(tt.item())
    rec = reconstruct_sharded(res, plan, ops, dist)
    realised = relative_error_sharded(x, rec, dist, ops=ops)
    del rec
    ok = abs(realised - res.relative_error) <= 1e-8
    if kind == "tolerance":
        ok = ok and realised <= param
    if not ok:
        raise SystemExit(f"bench: invalid sharded result: {realised} vs {res.relative_error}")
    # e2e: this rank's fibre block from pinned host memory every step, the
    # packed factors of its slices back to the host
    pinned = torch.empty(x.numel(), dtype=torch.float64, pin_memory=True)
    pinned.copy_(x)
    dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    d2h = 0
    for _ in range(args.steps):
        res = step(pinned.to(dev, non_blocking=True))
        u = res.u_data.cpu()
        g = res.g_data.cpu()
        d2h = (u.numel() + g.numel()) * 8
    torch.cuda.synchronize()
    te = torch.tensor([time.perf_counter() - t0], device=dev)
    dist.all_reduce(te, op=dist.ReduceOp.MAX)
    t_e2e = float(te.item())
    if rank == 0:
        import torch.cuda.nccl as tnccl
        try:
            nccl_version = ".".join(str(v) for v in tnccl.version())
        except Exception:
            nccl_version = None
        line = {
            "metric": metric_name(args.config), "value": args.steps * in_bytes / t_dev / 1e9,
            "unit": UNIT, "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * t_dev / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": f"synthetic ({args.config}, seed 0, one tensor sharded over the ranks)",
            "config": {"workload": f"{args.config}: {m}x{p}x{n} f64, {kind} {param}; fibre-sharded "
                                   "transform + NCCL all-to-all to slice ownership + all-gathered "
                                   "sigma, replicated threshold / energies",
                       "global_batch": 1, "seq_len": n, "parallelism": f"sharded x{world}"},
            "e2e": {"value": args.steps * in_bytes / t_e2e / 1e9, "unit": UNIT,
                    "h2d_bytes_per_step": in_bytes // world, "d2h_bytes_per_step": d2h,
                    "per": "rank 0 (every rank copies its own fibre block)"},
            "comm": {"backend": dist.get_backend(), "world_size": dist.get_world_size(),
                     "nccl": nccl_version,
                     "a2a_bytes_per_rank": in_bytes * (world - 1) // (world * world)},
            "clocks": clk.summary(), "gpu_launches": launches,
            "result": {"total_rank": int(res.ranks.sum()), "relative_error": res.relative_error,
                       "realised_error": realised},
        }
        emit(line)
    dist.barrier()
    dist.destroy_process_group()


def run_dry(args):
    """``--dry-run``: the launch plumbing alone on CPU (gloo): every rank
    joins the group, the world size and the sharded plan are checked, rank 0
    prints one JSON line.  No GPU and no compute."""
    import torch
    import torch.distributed as dist
    from paper_2605_16058_b200.sharded import ShardPlan
    rank, world, _ = dist_env()
    dist.init_process_group("gloo")
    dims = {"c1": (256, 256, 64), "c2": (361, 720, 1024), "c3": (1024, 1024, 512),
            "c4": (512, 512, 2048), "c5": (8192, 64, 4096), "c5t": (8192, 64, 4096)}[args.config]
    plan = ShardPlan(*dims, world, rank)
    counts = torch.tensor([plan.nf, plan.ns], dtype=torch.int64)
    dist.all_reduce(counts)
    if rank == 0:
        emit({"dry_run": True, "world_size": dist.get_world_size(), "config": args.config,
              "fibres": int(counts[0]), "slices": int(counts[1]),
              "mode": "replicas" if args.replicas else "sharded"})
    dist.barrier()
    dist.destroy_process_group()


_JSON_OUT = None   # the process's real stdout (fd 1 is pointed at stderr while the bench runs)


def emit(obj):
    """The one JSON line of this run, on the real stdout."""
    out = _JSON_OUT or sys.stdout
    out.write(json.dumps(obj) + "\n")
    out.flush()


def main():
    global _JSON_OUT
    args = parse()
    # stdout carries exactly one JSON line: libraries that print to fd 1 (the
    # NCCL version banner does, whatever NCCL_DEBUG_FILE says) land on stderr
    os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
    if not (args.gpus > 1 and "WORLD_SIZE" not in os.environ):   # (the relauncher just forwards its children)
        sys.stdout.flush()
        _JSON_OUT = os.fdopen(os.dup(1), "w")
        os.dup2(2, 1)
    _, world, _ = dist_env()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(relaunch_under_torchrun(args))
    if args.dry_run:
        run_dry(args)
    elif args.impl == "reference":
        run_reference(args)
    elif args.sharded or (world > 1 and not args.replicas):
        run_sharded(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
