"""t-SVDM compression entry points on the B200 (reference tsvdm.py).

Pipeline of ``tsvdm_tolerance`` for a tensor A (m x p x N slices):
  K1 forward transform (DCT: exact FFT + the reference operator's residual
     on tcgen05; other M: DMMA GEMM)
  ->  per-slice energies and the certified pruning (_tolerance_pruned):
      slices whose energy bounds every sigma^2 below the crossing value are
      left out of the SVD when the threshold certifies it
  ->  K3-K6 values pass (QR + band reduction, bulge chase, bisection) over
      the kept slices, keeping each slice's factorisation state
  ->  K7 device threshold (compute_threshold semantics; started at the
      left-out energy when pruned)
  ->  one small D2H (tau, energies, ranks total, certificate, SVD status)
  ->  K3-K6 truncated pass on the slices with rank > 0 from the kept state,
      writing the packed factors directly.
Everything stays in HBM; host inputs are uploaded once and outputs are
copied back once.
"""

from __future__ import annotations

import math
import os
import time
from contextlib import contextmanager
from dataclasses import dataclass
from math import prod

import numpy as np

from . import _native as nat
from .mode_product import (BATCHED, VARIANTS, DeferredResidual, deferrable, forward_device,
                           pipelined_upload_applies, upload_forward,
                           inverse_device)
from .slice_svd import (check_status, SLICES_PARALLEL, STRATEGIES, DeviceFactors, SliceSVDSet,
                        VariableRankFactors, pack_offsets_device, svd_full_device,
                        svd_truncated_device, svd_values_device)
from .tensors import DenseTensor, DeviceTensor, as_device
from .transform_set import CUSTOM, DATA_DRIVEN, TransformSet

__all__ = [
    "TRUNCATE", "COMPUTE_EFFICIENT", "MEMORY_EFFICIENT", "TOLERANCE_STRATEGIES",
    "METHOD_FIXED_RANK", "METHOD_TOLERANCE", "StageClock", "ThresholdResult",
    "compute_threshold", "TSVDMResult", "CompressedTensor", "starm_product", "full_tsvdm",
    "tsvdm_fixed_rank", "tsvdm_tolerance", "tsvdm_tolerance_stream", "reconstruct",
    "compression_ratio",
    "threshold_device", "relative_error_device", "reconstruct_fused",
]

TRUNCATE = "truncate"
COMPUTE_EFFICIENT = "compute-efficient"
MEMORY_EFFICIENT = "memory-efficient"
TOLERANCE_STRATEGIES = (TRUNCATE, COMPUTE_EFFICIENT, MEMORY_EFFICIENT)
METHOD_FIXED_RANK = "tsvdm1"
METHOD_TOLERANCE = "tsvdm2"


class StageClock:
    """Per-stage seconds (tsvdm.py:43-61).  On the device path each stage is
    bracketed by CUDA events on the current stream, resolved lazily when
    ``seconds`` is read, so timing adds no synchronisation."""

    def __init__(self):
        self._host = {}
        self._events = {}
        self.info = {}   # non-timing facts of the call (e.g. pruned slice count)

    @contextmanager
    def stage(self, name):
        import torch
        if torch.cuda.is_available():
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record()
            try:
                yield
            finally:
                b.record()
                self._events.setdefault(name, []).append((a, b))
        else:
            t0 = time.perf_counter()
            try:
                yield
            finally:
                self._host[name] = self._host.get(name, 0.0) + time.perf_counter() - t0

    def mark(self, name):
        self._host.setdefault(name, 0.0)

    @property
    def seconds(self):
        out = dict(self._host)
        for name, pairs in self._events.items():
            tot = 0.0
            for a, b in pairs:
                b.synchronize()
                tot += a.elapsed_time(b) / 1e3
            out[name] = out.get(name, 0.0) + tot
        return out


@dataclass
class ThresholdResult:
    """compute_threshold outcome (tsvdm.py:64-82)."""

    v: object
    w: object
    j: int
    tau: float
    ranks: object
    discarded_energy: float
    total_energy: float


def threshold_device(s_flat, r, n, epsilon, want_vw=False):
    """K7 on a device (r, N) column-major value matrix.  Returns device
    tensors (ranks, scal=[tau, discarded, total], j, v, w) -- asynchronous."""
    import torch
    dev = s_flat.device
    lib = nat.load()
    nbytes = lib.starm_threshold_workspace_bytes(r, n)
    ws = nat.workspace(nbytes, dev)
    ranks = torch.empty(n, dtype=torch.int64, device=dev)
    scal = torch.empty(3, dtype=torch.float64, device=dev)
    j = torch.empty(1, dtype=torch.int64, device=dev)
    v = torch.empty(r * n, dtype=torch.float64, device=dev) if want_vw else None
    w = torch.empty(r * n, dtype=torch.float64, device=dev) if want_vw else None
    nat.call("starm_threshold_f64", s_flat.data_ptr(), r, n, float(epsilon), nat.ptr(v),
             nat.ptr(w), ranks.data_ptr(), scal.data_ptr(), j.data_ptr(), ws.data_ptr(), nbytes,
             nat.stream_ptr(dev))
    return ranks, scal, j, v, w


def compute_threshold(s, epsilon) -> ThresholdResult:
    """Global energy threshold (tsvdm.py:85-115), run by the K7 kernels."""
    import torch
    epsilon = float(epsilon)
    if not 0.0 < epsilon < 1.0:
        raise ValueError(f"tolerance must lie in (0, 1), got {epsilon}")
    if isinstance(s, torch.Tensor) and not s.is_cuda:
        s = s.detach().numpy()   # host tensors take the host-array branch
    on_device = isinstance(s, torch.Tensor)
    if on_device:
        if s.dim() != 2:
            raise ValueError(f"expected an (r, N) value matrix, got {s.dim()} modes")
        if not bool(torch.isfinite(s).all()):
            raise ValueError("singular values must be finite")
        if s.numel() and bool((s < 0).any()):
            raise ValueError("singular values must be non-negative")
        r, n = s.shape
        flat = s.T.contiguous().reshape(-1).to(torch.float64)
    else:
        s = np.asarray(s, dtype=np.float64)
        if s.ndim != 2:
            raise ValueError(f"expected an (r, N) value matrix, got {s.ndim} modes")
        if not np.isfinite(s).all():
            raise ValueError("singular values must be finite")
        if s.size and s.min() < 0:
            raise ValueError("singular values must be non-negative")
        r, n = s.shape
        if s.size == 0:
            return ThresholdResult(np.zeros(0), np.zeros(0), 0, 0.0,
                                   np.zeros(n, dtype=np.int64), 0.0, 0.0)
        dev = nat.require_cuda()
        flat = torch.from_numpy(np.asfortranarray(s).reshape(-1, order="F").copy()).to(dev)
    ranks, scal, j, v, w = threshold_device(flat, r, n, epsilon, want_vw=True)
    sc = scal.cpu().numpy()
    jj = int(j.cpu().numpy()[0])
    if on_device:
        return ThresholdResult(v, w, jj, float(sc[0]), ranks, float(sc[1]), float(sc[2]))
    return ThresholdResult(v.cpu().numpy(), w.cpu().numpy(), jj, float(sc[0]),
                           ranks.cpu().numpy(), float(sc[1]), float(sc[2]))


@dataclass
class TSVDMResult:
    """Untruncated factorisation (tsvdm.py:118-130)."""

    factors: SliceSVDSet
    transforms: TransformSet
    dims: tuple

    def reconstruct(self, threads=1, ttm_variant=BATCHED):
        import torch
        f = self.factors
        host = isinstance(f.u, DenseTensor)
        dev = nat.require_cuda()
        m, p = self.dims[0], self.dims[1]
        n = prod(self.dims[2:])
        r = min(m, p)
        if host:
            s = torch.from_numpy(np.asfortranarray(f.s).reshape(-1, order="F").copy()).to(dev)
            u = as_device(f.u, dev).data
            v = as_device(f.v, dev).data
        else:
            s, u, v = f.s.T.contiguous().reshape(-1), f.u.data, f.v.data
            dev = u.device
        ranks = torch.full((n,), r, dtype=torch.int64, device=dev)
        u_off, g_off = pack_offsets_device(ranks, m, p)
        g = torch.empty(r * p * n, dtype=torch.float64, device=dev)
        st = nat.stream_ptr(dev)
        u_copy = torch.empty_like(u)  # pack writes U too; slice i's U block is already packed
        nat.call("starm_pack_from_full_f64", s.data_ptr(), u.data_ptr(), v.data_ptr(), m, p, n,
                 ranks.data_ptr(), u_off.data_ptr(), g_off.data_ptr(), u_copy.data_ptr(),
                 g.data_ptr(), st)
        chat = DeviceTensor.empty(self.dims, dev)
        nat.call("starm_unpack_facewise_f64", u.data_ptr(), g.data_ptr(), ranks.data_ptr(),
                 u_off.data_ptr(), g_off.data_ptr(), m, p, n, chat.data.data_ptr(), st)
        out = inverse_device(chat, self.transforms)
        return out.to_host() if host else out


@dataclass
class CompressedTensor:
    """Packed variable-rank factors + transforms + shape (tsvdm.py:132-182).
    ``factors`` is a VariableRankFactors (host) or DeviceFactors (HBM)."""

    dims: tuple
    transforms: TransformSet
    factors: object
    method: str
    param: float
    discarded_energy: float | None = None
    total_energy: float | None = None

    def __post_init__(self):
        self.dims = tuple(int(n) for n in self.dims)
        if len(self.dims) < 3:
            raise ValueError("compressed tensors have at least three modes")
        if self.method not in (METHOD_FIXED_RANK, METHOD_TOLERANCE):
            raise ValueError(f"unknown method {self.method!r}")
        self.transforms.check_dims(self.dims)
        f = self.factors
        if (f.slice_rows, f.slice_cols) != (self.dims[0], self.dims[1]):
            raise ValueError(f"factor slices are {f.slice_rows}x{f.slice_cols}, "
                             f"tensor slices are {self.dims[0]}x{self.dims[1]}")
        if f.num_slices != prod(self.dims[2:]):
            raise ValueError(f"{f.num_slices} factor slices for {prod(self.dims[2:])} tensor slices")
        if self.method == METHOD_FIXED_RANK and isinstance(f, VariableRankFactors):
            r = int(self.param)
            if f.ranks.size and not (f.ranks == r).all():
                raise ValueError("fixed-rank artifacts must have one uniform rank")

    @property
    def ranks(self) -> np.ndarray:
        return self.factors.ranks

    def relative_error(self):
        if self.discarded_energy is None or self.total_energy is None:
            return None
        if self.total_energy == 0.0:
            return 0.0
        return math.sqrt(self.discarded_energy / self.total_energy)

    def to_host(self) -> "CompressedTensor":
        return CompressedTensor(self.dims, self.transforms, self.factors.to_host(), self.method,
                                self.param, self.discarded_energy, self.total_energy)


def _check_decomposable(t):
    if len(t.dims) < 3:
        raise ValueError("decompositions apply to tensors with at least three modes")


def _check_threads(threads):
    if int(threads) < 1:
        raise ValueError(f"thread count must be positive, got {threads}")


def _check_common(threads, svd_strategy, ttm_variant):
    _check_threads(threads)
    if svd_strategy not in STRATEGIES:
        raise ValueError(f"unknown slice SVD strategy {svd_strategy!r}")
    if ttm_variant not in VARIANTS:
        raise ValueError(f"unknown ttm variant {ttm_variant!r}")


def starm_product(a, b, ts: TransformSet, ttm_variant=BATCHED, threads=1):
    """A *_M B (tsvdm.py:219-233): forward TTMs, facewise DMMA GEMM, inverse TTMs."""
    _check_decomposable(a)
    _check_threads(threads)
    if ttm_variant not in VARIANTS:
        raise ValueError(f"unknown ttm variant {ttm_variant!r}")
    if len(a.dims) != len(b.dims) or tuple(a.dims[2:]) != tuple(b.dims[2:]):
        raise ValueError(f"trailing dims differ: {a.dims} vs {b.dims}")
    if a.dims[1] != b.dims[0]:
        raise ValueError(f"slice shapes {a.dims[:2]} and {b.dims[:2]} do not chain")
    ts.check_dims(a.dims)
    host = isinstance(a, DenseTensor)
    dev = nat.require_cuda() if host else a.device
    ahat = upload_forward(a, ts, dev)
    bhat = forward_device(as_device(b, dev), ts)
    m, p, cols = a.dims[0], a.dims[1], b.dims[1]
    n = prod(a.dims[2:])
    out_dims = (m, cols) + tuple(a.dims[2:])
    chat = DeviceTensor.empty(out_dims, dev)
    nat.call("starm_facewise_gemm_f64", ahat.data.data_ptr(), bhat.data.data_ptr(),
             chat.data.data_ptr(), m, p, cols, n, nat.stream_ptr(dev))
    out = inverse_device(chat, ts)
    return out.to_host() if host else out


def full_tsvdm(a, ts: TransformSet, threads=1, svd_strategy=SLICES_PARALLEL,
               ttm_variant=BATCHED) -> TSVDMResult:
    """Every transform-domain slice factored (tsvdm.py:236-243)."""
    from .slice_svd import svd_all_slices
    _check_decomposable(a)
    _check_common(threads, svd_strategy, ttm_variant)
    ts.check_dims(a.dims)
    host = isinstance(a, DenseTensor)
    dev = nat.require_cuda() if host else a.device
    ahat = upload_forward(a, ts, dev)
    factors = svd_all_slices(ahat.to_host() if host else ahat)
    return TSVDMResult(factors, ts, tuple(a.dims))


def _finish(a, ts, factors, method, param, discarded, total, host):
    if host:
        factors = factors.to_host()
    return CompressedTensor(tuple(a.dims), ts, factors, method, param, discarded, total)


def _resolve_devices(devices):
    """``devices`` of the drop-in entry points (SURVEY 8b "add devices="):
    None -> the current CUDA device; an int / str / torch.device -> that
    device; a torch.distributed ProcessGroup or the string "dist" (the
    default group) -> the sharded multi-GPU pipeline over that group's ranks
    (one process per GPU).  Returns (device or None, group or None)."""
    import torch
    if devices is None:
        return None, None
    if isinstance(devices, str) and devices == "dist":
        import torch.distributed as dist
        return None, dist.group.WORLD
    if isinstance(devices, (int, str, torch.device)):
        return nat.require_cuda(devices if not isinstance(devices, int) else f"cuda:{devices}"), None
    if type(devices).__name__ == "ProcessGroup":
        return None, devices
    raise ValueError(f"devices must be None, a CUDA device, 'dist' or a ProcessGroup, got {devices!r}")


def _sharded_call(a, ts, group, kind, param):
    """SPMD drop-in over a process group: every rank passes the same (full)
    host tensor, takes its fibre block, runs sharded.py's pipeline (fibre
    transform, NCCL all-to-all to slice ownership, replicated threshold /
    energies), and gets the full CompressedTensor (factors all-gathered)."""
    import torch
    import torch.distributed as dist
    from .sharded import (DeviceOps, ShardPlan, gather_factors, scatter_fibres,
                          tsvdm_fixed_rank_sharded, tsvdm_tolerance_sharded)
    if len(a.dims) != 3 or len(ts) != 1:
        raise ValueError("the sharded pipeline handles 3-way tensors (one transform)")
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    dev = nat.require_cuda()
    m, p, n = a.dims
    plan = ShardPlan(m, p, n, world, rank)
    host = isinstance(a, DenseTensor)
    arr = a.array if host else a.to_host().array
    local = torch.from_numpy(scatter_fibres(arr, plan).reshape(-1, order="F").copy()).to(dev)
    ops = DeviceOps(ts[0], dev)
    if kind == METHOD_FIXED_RANK:
        res = tsvdm_fixed_rank_sharded(local, plan, ops, int(param), dist, group)
    else:
        res = tsvdm_tolerance_sharded(local, plan, ops, float(param), dist, group)
    u, g = gather_factors(res, plan, dist, group)
    ranks = torch.from_numpy(np.ascontiguousarray(res.ranks)).to(dev)
    u_off, g_off = pack_offsets_device(ranks, m, p)
    total = int(res.ranks.sum())
    factors = DeviceFactors(m, p, ranks, u_off, g_off, u, g, total)
    factors._host_ranks = np.asarray(res.ranks, dtype=np.int64)
    return _finish(a, ts, factors, kind, float(param), res.discarded_energy, res.total_energy,
                   host)


def tsvdm_fixed_rank(a, ts: TransformSet, rank, threads=1, svd_strategy=SLICES_PARALLEL,
                     ttm_variant=BATCHED, devices=None) -> CompressedTensor:
    """Uniform rank per slice (tsvdm.py:246-265).  ``devices``: see
    _resolve_devices (a process group runs the sharded multi-GPU pipeline)."""
    import torch
    _check_decomposable(a)
    ts.check_dims(a.dims)
    m, p = a.dims[0], a.dims[1]
    rank = int(rank)
    if not 1 <= rank <= min(m, p):
        raise ValueError(f"rank must lie in [1, {min(m, p)}], got {rank}")
    _check_common(threads, svd_strategy, ttm_variant)
    want, group = _resolve_devices(devices)
    if group is not None:
        return _sharded_call(a, ts, group, METHOD_FIXED_RANK, rank)
    host = isinstance(a, DenseTensor)
    dev = (want or nat.require_cuda()) if host else a.device
    n = prod(a.dims[2:])
    r = min(m, p)
    ahat = upload_forward(a, ts, dev)
    ahat3 = DeviceTensor(ahat.data, (m, p, n))
    ranks = torch.full((n,), rank, dtype=torch.int64, device=dev)
    factors, s = svd_truncated_device(ahat3, ranks, rank * n, keep_values=True)
    factors._host_ranks = np.full(n, rank, dtype=np.int64)
    en = torch.empty(2, dtype=torch.float64, device=dev)
    nat.call("starm_tail_energy_f64", s.data_ptr(), r, n, rank, en.data_ptr(), nat.stream_ptr(dev))
    d, t = en.cpu().numpy()
    return _finish(a, ts, factors, METHOD_FIXED_RANK, float(rank), float(d), float(t), host)


def tsvdm_tolerance(a, ts: TransformSet, epsilon, strategy=MEMORY_EFFICIENT, threads=1,
                    svd_strategy=SLICES_PARALLEL, ttm_variant=BATCHED, clock=None, devices=None):
    """Global-threshold ranks (tsvdm.py:268-321).  All three strategies give
    identical ranks and factors; on the device ``memory-efficient`` and
    ``compute-efficient`` are the same two-pass schedule (the transform-domain
    tensor already stays resident in HBM), ``truncate`` factors every slice
    fully and packs from the full factors.  ``devices``: see _resolve_devices
    (a process group runs the sharded multi-GPU pipeline)."""
    import torch
    _check_decomposable(a)
    ts.check_dims(a.dims)
    epsilon = float(epsilon)
    if not 0.0 < epsilon < 1.0:
        raise ValueError(f"tolerance must lie in (0, 1), got {epsilon}")
    if strategy not in TOLERANCE_STRATEGIES:
        raise ValueError(f"unknown tolerance strategy {strategy!r}")
    _check_common(threads, svd_strategy, ttm_variant)
    clock = clock if clock is not None else StageClock()
    want, group = _resolve_devices(devices)
    if group is not None:
        return _sharded_call(a, ts, group, METHOD_TOLERANCE, epsilon)
    host = isinstance(a, DenseTensor)
    dev = (want or nat.require_cuda()) if host else a.device
    m, p = a.dims[0], a.dims[1]
    n = prod(a.dims[2:])
    r = min(m, p)
    deferred = None
    if PRUNE and strategy != TRUNCATE and deferrable(ts, a.dims):
        # exact FFT DCT now; the reference operator's residual is added to the
        # slices the pruning keeps (or to all of them if it does not prune)
        if pipelined_upload_applies(a, ts):
            # host input: block-wise H2D with the DCT, operand rows and slice
            # energies of each block running behind the next block's copy
            deferred = DeferredResidual.from_host(a, ts[0], dev)
        else:
            deferred = DeferredResidual(as_device(a, dev), ts[0])
        ahat = deferred.out
    else:
        ahat = upload_forward(a, ts, dev)
    ahat3 = DeviceTensor(ahat.data, (m, p, n))
    if strategy == TRUNCATE:
        with clock.stage("stage1-svd"):
            s, u, v = svd_full_device(ahat3)
        with clock.stage("threshold"):
            ranks, scal, j, _, _ = threshold_device(s, r, n, epsilon)
            summary = _summary(ranks, scal)
        clock.mark("stage2-svd")
        with clock.stage("pack"):
            total_rank = summary[3]
            u_off, g_off = pack_offsets_device(ranks, m, p)
            u_data = torch.empty(max(total_rank * m, 1), dtype=torch.float64, device=dev)
            g_data = torch.empty(max(total_rank * p, 1), dtype=torch.float64, device=dev)
            nat.call("starm_pack_from_full_f64", s.data_ptr(), u.data_ptr(), v.data_ptr(), m, p, n,
                     ranks.data_ptr(), u_off.data_ptr(), g_off.data_ptr(), u_data.data_ptr(),
                     g_data.data_ptr(), nat.stream_ptr(dev))
            factors = DeviceFactors(m, p, ranks, u_off, g_off, u_data[: total_rank * m],
                                    g_data[: total_rank * p], total_rank)
    else:
        pruned = _tolerance_pruned(ahat3, epsilon, strategy, clock, deferred) if PRUNE else None
        if pruned is not None:
            factors, discarded, total = pruned
            return _finish(a, ts, factors, METHOD_TOLERANCE, epsilon, discarded, total, host)
        if deferred is not None:
            deferred.apply_all()     # unpruned: every slice gets the reference operator
        # Keep every slice's factorisation in HBM between the passes when it
        # fits comfortably (always for compute-efficient); otherwise refactor
        # the rank>0 slices (memory-efficient in the reference's sense).
        keep = strategy == COMPUTE_EFFICIENT or _state_fits(ahat3)
        pending = []  # device status pairs, read back with the next D2H
        with clock.stage("stage1-svd"):
            if keep:
                s, state = svd_values_device(ahat3, keep_state=True, defer=pending)
            else:
                s, state = svd_values_device(ahat3, defer=pending), None
        with clock.stage("threshold"):
            ranks, scal, j, _, _ = threshold_device(s, r, n, epsilon)
            summary = _summary(ranks, scal, pending)
        pending = []
        with clock.stage("stage2-svd"):
            factors, _ = svd_truncated_device(ahat3, ranks, summary[3], state=state, defer=pending)
            if pending:
                check_status(torch.cat(pending).cpu().numpy())
        del state
        clock.mark("pack")
    tau, discarded, total, _ = summary
    return _finish(a, ts, factors, METHOD_TOLERANCE, epsilon, discarded, total, host)


def tsvdm_tolerance_stream(tensors, ts: TransformSet, epsilon, strategy=MEMORY_EFFICIENT,
                           device=None):
    """Compress a sequence of host tensors (DenseTensor, same transform set)
    with ``tsvdm_tolerance``, yielding one host CompressedTensor per input in
    order.  The host-to-device copy of tensor k+1 runs on a copy stream while
    tensor k is compressed (two device input buffers, event-ordered reuse),
    so for pinned inputs a stream of tensors costs ~max(copy, compute) per
    tensor instead of copy + compute.  Results are identical to calling
    ``tsvdm_tolerance`` on each tensor."""
    import torch
    dev = nat.require_cuda(device)
    copy_stream = torch.cuda.Stream(dev)
    bufs, ready, free, keep = [None, None], [None, None], [None, None], [None, None]

    def issue(t, b):
        if not isinstance(t, DenseTensor):
            raise TypeError(f"expected DenseTensor inputs, got {type(t).__name__}")
        ts.check_dims(t.dims)
        src = torch.from_numpy(np.ascontiguousarray(t.data))
        compute = torch.cuda.current_stream(dev)
        with torch.cuda.stream(copy_stream):
            if bufs[b] is None or bufs[b].numel() != src.numel():
                # allocated on the copy stream (its first writer) and ordered
                # after everything already queued on the compute stream, so a
                # block freed by in-flight compute work is never overwritten;
                # the compute stream's later use is recorded for the allocator
                copy_stream.wait_stream(compute)
                bufs[b] = torch.empty(src.numel(), dtype=torch.float64, device=dev)
                bufs[b].record_stream(compute)
            if free[b] is not None:
                copy_stream.wait_event(free[b])
            bufs[b].copy_(src, non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(copy_stream)
        ready[b], keep[b] = ev, src

    it = iter(tensors)
    cur = next(it, None)
    if cur is None:
        return
    issue(cur, 0)
    b = 0
    while cur is not None:
        nxt = next(it, None)
        if nxt is not None:
            issue(nxt, 1 - b)  # overlaps the compression of ``cur``
        torch.cuda.current_stream(dev).wait_event(ready[b])
        c = tsvdm_tolerance(DeviceTensor(bufs[b], cur.dims), ts, epsilon, strategy)
        ev = torch.cuda.Event()
        ev.record(torch.cuda.current_stream(dev))
        free[b] = ev
        yield c.to_host()
        cur, b = nxt, 1 - b


PRUNE = os.environ.get("STARM_PRUNE", "1") != "0"   # STARM_PRUNE=0: diagnostic, unpruned
PRUNE_REFINE = os.environ.get("STARM_PRUNE_REFINE", "1") != "0"   # 0: the plain energy rule only
PRUNE_GAMMA = 0.3      # left-out energy target as a fraction of the budget
PRUNE_MIN = 0.25       # prune only when at least this fraction of the slices drops out


def prune_select(ahat3, epsilon):
    """The slice selection the pruned tolerance path tries first (see
    prune_plan): (kept slice ids ascending, e0 = left-out energy, tbound =
    bound on every left-out sigma^2) or None when nothing prunes."""
    plan = prune_plan(ahat3, epsilon)
    return plan[0] if plan else None


def prune_choose(f, epsilon):
    """Host half of prune_select on the per-slice energies ``f`` (also used by
    the sharded path on all-reduced energies, so every rank chooses the same
    slices): (kept ids ascending, e0, tbound) or None."""
    f = np.asarray(f, dtype=np.float64)
    n = f.size
    if n < 8 or not np.isfinite(f).all():
        return None                      # the SVD names the non-finite slice
    # (numpy's pairwise sums: deterministic for a given f, so every rank of the
    # sharded path derives the same numbers; math.fsum cost 0.1 ms per call here)
    budget = epsilon * epsilon * float(np.sum(f))
    order = np.argsort(f, kind="stable")
    k = int(np.searchsorted(np.cumsum(f[order]), PRUNE_GAMMA * budget, side="right"))
    if k < PRUNE_MIN * n or k >= n:
        return None
    keep_ids = np.sort(order[k:])
    return keep_ids, float(np.sum(f[np.sort(order[:k])])), float(f[order[k - 1]])


PRUNE_GAMMA2 = 0.4      # left-out energy cap once the marginal slices carry the sharper bound
PRUNE_REFINE_MAX = 64   # at most this many marginal slices get the sharper bound
PRUNE_CLUSTER_SLICES = None   # kept-slice count the refinement aims for (None: half the SMs)


def prune_refine(ahat3, f, epsilon, sel):
    """A second, sharper selection on top of ``sel`` = prune_choose(f): the
    kept slices of smallest energy are often rank-0 slices whose energy is
    spread over two or more comparable singular values (c2: sine / cosine
    pairs, sigma_1^2 ~ f / 2), so f overstates their sigma_max^2.  For the
    marginal ones (ascending f while the left-out energy stays below
    PRUNE_GAMMA2 of the budget) compute b_i = ||G_i^2||_F^(1/2) with G_i the
    slice's Gram matrix: (sum sigma^8)^(1/4) >= sigma_1^2, two small batched
    DMMA products per slice (starm_facewise_gemm_f64, starm_slice_energy_f64).
    A marginal slice whose b_i does not exceed the bound ``tbound`` that
    ``sel`` already certifies against is left out too: tbound is unchanged,
    only e0 grows.  Worth doing only when it brings the kept count down to
    half the SMs or fewer, where the reduce kernel puts a cluster of CTAs on
    each slice.  Returns (keep_ids, e0, tbound) or None."""
    import torch
    keep_ids, e0, tbound = sel
    m, p, n = ahat3.dims
    dev = ahat3.device
    half = PRUNE_CLUSTER_SLICES or torch.cuda.get_device_properties(dev).multi_processor_count // 2
    if keep_ids.size <= half:
        return None
    f = np.asarray(f, dtype=np.float64)
    budget = epsilon * epsilon * float(f.sum())      # (a cap for a heuristic: plain summation will do)
    fk = f[keep_ids]
    ordk = keep_ids[np.argsort(fk, kind="stable")[:PRUNE_REFINE_MAX + 1]]
    cum = e0 + np.cumsum(f[ordk])
    nc = int(np.searchsorted(cum, PRUNE_GAMMA2 * budget, side="right"))
    if nc == 0 or nc > PRUNE_REFINE_MAX or keep_ids.size - nc > half:
        return None
    if nc * (2 * m * p + 2 * min(m, p) ** 2) * 8 > (2 << 30):
        return None                      # (the bound's scratch is capped at 2 GB)
    cand = np.sort(ordk[:nc])
    ids = torch.from_numpy(cand.astype(np.int64)).to(dev)
    a = ahat3.data.view(n, p, m).index_select(0, ids)            # column-major m x p slices
    at = a.transpose(1, 2).contiguous()                          # column-major p x m: the transposes
    q = min(m, p)
    g = torch.empty(nc * q * q, dtype=torch.float64, device=dev)
    st = nat.stream_ptr(dev)
    if m <= p:   # G = A A^T (m x m)
        nat.call("starm_facewise_gemm_f64", a.data_ptr(), at.data_ptr(), g.data_ptr(), m, p, m, nc, st)
    else:        # G = A^T A (p x p)
        nat.call("starm_facewise_gemm_f64", at.data_ptr(), a.data_ptr(), g.data_ptr(), p, m, p, nc, st)
    g2 = torch.empty_like(g)
    nat.call("starm_facewise_gemm_f64", g.data_ptr(), g.data_ptr(), g2.data_ptr(), q, q, q, nc, st)
    e8 = torch.empty(nc, dtype=torch.float64, device=dev)
    nat.call("starm_slice_energy_f64", g2.data_ptr(), q * q, nc, e8.data_ptr(), st)
    # (sum sigma^8)^(1/4), widened well past the products' rounding
    b = np.sqrt(np.sqrt(e8.cpu().numpy())) * (1.0 + 1e-9)
    drop = cand[np.isfinite(b) & (b <= tbound)]
    if drop.size == 0 or keep_ids.size - drop.size > half:
        return None
    keep2 = keep_ids[~np.isin(keep_ids, drop)]
    # e0 of the larger left-out set, summed exactly like prune_choose's
    mask = np.ones(n, dtype=bool)
    mask[keep2] = False
    return keep2, float(np.sum(f[mask])), tbound


def _tolerance_pruned(ahat3, epsilon, strategy, clock, deferred=None):
    """Certified slice pruning for tsvdm_tolerance (same ranks, factors and
    energies as the unpruned path, which the reference computes).

    Every sigma^2 of slice i is at most f_i = ||Ahat_i||_F^2.  Leave out the
    slices of smallest f whose total energy e0 stays below PRUNE_GAMMA of the
    budget eps^2 * sum(f); t = their largest f.  The values pass, threshold
    and truncated pass then run on the remaining slices only, with the
    threshold's running sum started at e0 (starm_threshold_pruned_f64).  If
    the crossing value lies above t, every value <= t -- in particular every
    left-out sigma^2 -- is discarded by compute_threshold's rule
    (tsvdm.py:85-115) whatever its exact size: the left-out slices have rank
    0, the others get the reference's ranks, the discarded energy is e0 plus
    their dropped squares.  Otherwise (certificate fails) return None and the
    caller runs the unpruned path.  Returns (factors, discarded, total)."""
    import torch
    m, p, n = ahat3.dims
    r = min(m, p)
    dev = ahat3.device
    if n < 8 or strategy not in (MEMORY_EFFICIENT, COMPUTE_EFFICIENT):
        return None
    with clock.stage("prune-energy"):
        sels = prune_plan(ahat3, epsilon, deferred.energies if deferred is not None else None)
    # the sharper selection first; if its certificate fails the plain one
    # (one more values pass over a single wave), then the unpruned path
    for sel in sels:
        res = _pruned_attempt(ahat3, epsilon, strategy, clock, deferred, sel)
        if res is not None:
            return res
    return None


def prune_plan(ahat3, epsilon, f_dev=None):
    """The selections the pruned tolerance path tries, in order: the sharper
    one (prune_refine) when it applies, then the plain energy rule
    (prune_choose); [] when nothing prunes."""
    import torch
    m, p, n = ahat3.dims
    if f_dev is None:
        f_dev = torch.empty(n, dtype=torch.float64, device=ahat3.device)
        nat.call("starm_slice_energy_f64", ahat3.data.data_ptr(), m * p, n, f_dev.data_ptr(),
                 nat.stream_ptr(ahat3.device))
    f = f_dev.cpu().numpy()
    sel = prune_choose(f, epsilon)
    if sel is None:
        return []
    sharp = prune_refine(ahat3, f, epsilon, sel) if PRUNE_REFINE else None
    return [sharp, sel] if sharp is not None else [sel]


def _pruned_attempt(ahat3, epsilon, strategy, clock, deferred, sel):
    """One pruned computation with the selection ``sel``; None when its
    certificate fails."""
    import torch
    m, p, n = ahat3.dims
    r = min(m, p)
    dev = ahat3.device
    keep_ids, e0, tbound = sel
    if deferred is not None:
        # energies of the exact-DCT slices: the reference operator differs by
        # |Delta x| ~ 1e-13 |x|, so widen the bound well past that
        tbound *= 1.0 + 1e-9
    k = n - int(keep_ids.size)
    ns = int(keep_ids.size)
    ids_dev = torch.from_numpy(keep_ids.astype(np.int64)).to(dev)
    sub = DeviceTensor(ahat3.data.view(n, m * p).index_select(0, ids_dev).reshape(-1), (m, p, ns))
    if deferred is not None:
        deferred.apply_cols(sub.data, ids_dev)   # reference operator on the kept slices only
    pending = []
    with clock.stage("stage1-svd"):
        keep = strategy == COMPUTE_EFFICIENT or _state_fits(sub)
        if keep:
            s, state = svd_values_device(sub, keep_state=True, defer=pending)
        else:
            s, state = svd_values_device(sub, defer=pending), None
    with clock.stage("threshold"):
        lib = nat.load()
        nbytes = lib.starm_threshold_workspace_bytes(r, ns)
        ws = nat.workspace(nbytes, dev)
        ranks_s = torch.empty(ns, dtype=torch.int64, device=dev)
        scal = torch.empty(3, dtype=torch.float64, device=dev)
        j = torch.empty(1, dtype=torch.int64, device=dev)
        cert = torch.empty(1, dtype=torch.int32, device=dev)
        nat.call("starm_threshold_pruned_f64", s.data_ptr(), r, ns, float(epsilon), e0, tbound,
                 ranks_s.data_ptr(), scal.data_ptr(), j.data_ptr(), cert.data_ptr(), ws.data_ptr(),
                 nbytes, nat.stream_ptr(dev))
        h = torch.cat([scal, ranks_s.sum().reshape(1).to(torch.float64),
                       cert.to(torch.float64)] + [st.to(torch.float64) for st in pending])
        h = h.cpu().numpy()
        if pending:
            check_status(h[5:].astype(np.int64))
    clock.info["pruned_slices"] = k
    if h[4] != 1.0:
        clock.info["prune_certificate"] = "failed"
        return None
    clock.info["prune_certificate"] = "ok"
    _, discarded, total, total_rank = float(h[0]), float(h[1]), float(h[2]), int(h[3])
    with clock.stage("stage2-svd"):
        pending = []
        fs, _ = svd_truncated_device(sub, ranks_s, total_rank, state=state, defer=pending)
        if pending:
            check_status(torch.cat(pending).cpu().numpy())
        del state
        ranks = torch.zeros(n, dtype=torch.int64, device=dev)
        ranks.index_copy_(0, ids_dev, ranks_s)
        u_off, g_off = pack_offsets_device(ranks, m, p)
        # the kept slices are in ascending slice order and the left-out ones
        # have rank 0, so the subset's packed payload IS the global layout
        factors = DeviceFactors(m, p, ranks, u_off, g_off, fs.u_data, fs.g_data, total_rank)
    return factors, discarded, total


_HBM_BUDGET = {}  # device index -> bytes this process can hold (free + own reserved), read once


def _state_fits(x) -> bool:
    """True when the per-slice SVD state needs < 1/4 of the free HBM.

    cudaMemGetInfo occasionally blocks for tens of milliseconds, so it is
    queried once per device; later calls subtract this process's current
    allocations from that budget."""
    import torch
    from .slice_svd import state_bytes
    idx = x.device.index if x.device.index is not None else torch.cuda.current_device()
    if idx not in _HBM_BUDGET:
        free, _ = torch.cuda.mem_get_info(x.device)
        _HBM_BUDGET[idx] = free + torch.cuda.memory_reserved(x.device)
    free = _HBM_BUDGET[idx] - torch.cuda.memory_allocated(x.device)
    return state_bytes(x) < free // 4


def _summary(ranks, scal, pending=()):
    """One small D2H: (tau, discarded, total, sum of ranks) plus any deferred
    SVD status pairs, which are checked here."""
    import torch
    parts = [scal, ranks.sum().reshape(1).to(torch.float64)]
    parts += [st.to(torch.float64) for st in pending]
    h = torch.cat(parts).cpu().numpy()
    if pending:
        check_status(h[4:].astype(np.int64))
    return float(h[0]), float(h[1]), float(h[2]), int(h[3])


def _device_factors(c: CompressedTensor, dev):
    import torch
    f = c.factors
    if isinstance(f, DeviceFactors):
        return f
    ranks = torch.from_numpy(np.ascontiguousarray(f.ranks)).to(dev)
    u_off, g_off = pack_offsets_device(ranks, f.slice_rows, f.slice_cols)
    u = torch.from_numpy(f.u_data).to(dev) if f.u_data.size else torch.empty(1, dtype=torch.float64, device=dev)
    g = torch.from_numpy(f.g_data).to(dev) if f.g_data.size else torch.empty(1, dtype=torch.float64, device=dev)
    return DeviceFactors(f.slice_rows, f.slice_cols, ranks, u_off, g_off, u, g, f.total_rank)


def _fused_operator(c: CompressedTensor, nnz, dev):
    """Row-major inverse operator for starm_reconstruct_f64, or None when the
    unfused path is cheaper: 3-way tensors only; the identity is a copy; the
    DCT's FFT route costs ~2 passes over the tensor, so the K = nnz dense
    product wins only while nnz is small against n."""
    from .transform_set import DCT, IDENTITY
    if len(c.dims) != 3 or len(c.transforms) != 1:
        return None
    tr = c.transforms[0]
    n = c.dims[2]
    if tr.kind == IDENTITY:
        return None
    if tr.kind == DCT and nnz > max(16, n // 8):
        return None
    return tr.device_operand(dev, transpose=True)   # M^T, row-major (ttm.py:147-153)


def reconstruct_fused(c: CompressedTensor, a=None, dev=None, minv=None):
    """K9 + inverse transform + K10 in one C-ABI call (starm_reconstruct_f64):
    returns (reconstruction DeviceTensor, relative error or None).  ``minv``
    overrides the inverse operator (row-major n x n, e.g. an explicit M^-1);
    raises ValueError when the fused form does not apply (d-way tensors)."""
    import torch
    f = c.factors
    if dev is None:
        dev = f.u_data.device if isinstance(f, DeviceFactors) else nat.require_cuda()
    df = _device_factors(c, dev)
    m, p = c.dims[0], c.dims[1]
    if len(c.dims) != 3:
        raise ValueError("the fused reconstruction applies to 3-way tensors")
    n = c.dims[2]
    nz = torch.nonzero(df.ranks_dev > 0).reshape(-1).to(torch.int64)
    nnz = int(nz.numel())
    op = minv if minv is not None else _fused_operator(c, nnz, dev)
    if op is None:
        from .transform_set import IDENTITY
        if len(c.transforms) == 1 and c.transforms[0].kind != IDENTITY:
            op = c.transforms[0].device_operand(dev, transpose=True)
        else:
            raise ValueError("no dense inverse operator for the fused reconstruction")
    if not isinstance(op, torch.Tensor):
        op = torch.from_numpy(np.ascontiguousarray(op, dtype=np.float64)).to(dev)
    lib = nat.load()
    nbytes = lib.starm_reconstruct_workspace_bytes(m, p, n, nnz)
    ws = nat.workspace(nbytes, dev)
    out = DeviceTensor.empty(c.dims, dev)
    err2 = torch.empty(2, dtype=torch.float64, device=dev) if a is not None else None
    nat.call("starm_reconstruct_f64", df.u_data.data_ptr(), df.g_data.data_ptr(),
             df.ranks_dev.data_ptr(), df.u_off.data_ptr(), df.g_off.data_ptr(), m, p, n,
             nz.data_ptr() if nnz else 0, nnz, op.data_ptr(),
             a.data.data_ptr() if a is not None else 0, out.data.data_ptr(), nat.ptr(err2),
             ws.data_ptr(), nbytes, nat.stream_ptr(dev))
    if a is None:
        return out, None
    d2, a2 = err2.cpu().numpy()
    return out, (math.sqrt(d2 / a2) if a2 > 0 else 0.0)


def reconstruct_device(c: CompressedTensor, dev=None) -> DeviceTensor:
    f = c.factors
    if dev is None:
        dev = f.u_data.device if isinstance(f, DeviceFactors) else nat.require_cuda()
    df = _device_factors(c, dev)
    m, p = c.dims[0], c.dims[1]
    n = prod(c.dims[2:])
    if len(c.dims) == 3:
        nnz = int((df.ranks_dev > 0).sum().item())
        if _fused_operator(c, nnz, dev) is not None:
            return reconstruct_fused(c, dev=dev)[0]
    chat = DeviceTensor.empty(c.dims, dev)
    nat.call("starm_unpack_facewise_f64", df.u_data.data_ptr(), df.g_data.data_ptr(),
             df.ranks_dev.data_ptr(), df.u_off.data_ptr(), df.g_off.data_ptr(), m, p, n,
             chat.data.data_ptr(), nat.stream_ptr(dev))
    return inverse_device(chat, c.transforms)


def reconstruct(c: CompressedTensor, threads=1, ttm_variant=BATCHED):
    """Dense tensor from packed factors (tsvdm.py:342-357)."""
    _check_threads(threads)
    if ttm_variant not in VARIANTS:
        raise ValueError(f"unknown ttm variant {ttm_variant!r}")
    out = reconstruct_device(c)
    return out if isinstance(c.factors, DeviceFactors) else out.to_host()


def relative_error_device(a: DeviceTensor, b: DeviceTensor) -> float:
    """||a - b|| / ||a|| with the K10 deterministic reduction."""
    import torch
    dev = a.device
    lib = nat.load()
    nbytes = lib.starm_error_sums_workspace_bytes(a.size)
    ws = nat.workspace(nbytes, dev)
    out = torch.empty(2, dtype=torch.float64, device=dev)
    nat.call("starm_error_sums_f64", a.data.data_ptr(), b.data.data_ptr(), a.size, out.data_ptr(),
             ws.data_ptr(), nbytes, nat.stream_ptr(dev))
    d2, a2 = out.cpu().numpy()
    return math.sqrt(d2 / a2) if a2 > 0 else 0.0


def compression_ratio(c: CompressedTensor) -> float:
    """Original entries / stored entries (tsvdm.py:360-372)."""
    m, p = c.dims[0], c.dims[1]
    stored = c.factors.total_rank * (m + p)
    stored += sum(t.size ** 2 for t in c.transforms if t.kind in (DATA_DRIVEN, CUSTOM))
    if stored == 0:
        return math.inf
    return prod(c.dims) / stored
