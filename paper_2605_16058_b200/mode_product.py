"""Mode-k tensor-times-matrix on the B200 (reference ttm.py).

Every variant of the reference (``batched`` / ``loop`` / ``parfor``,
ttm.py:113-135) is one launch of the FP64 DMMA GEMM kernel here: the
column-major buffer is ``batch`` row-major (inner x rows) blocks and the
kernel computes dst[b] = M @ src[b] for all b in a single grid.  The
variant and thread arguments are validated exactly like the reference and
then have no further effect.

Structured transforms apply the SAME operator as the reference's dense
product, faster.  The identity kind is a device copy (the product with I is
exact).  The DCT kind with a power-of-two extent in [256, 4096] whose stored
matrix is within 1e-9 of the exact DCT-II (always, for dct_matrix) runs the
O(n log n) FFT DCT-II / DCT-III kernel (starm_dct_f64) for the exact
transform and then adds the reference matrix's own rounding, Delta =
M - M_exact, with a tcgen05 bf16 GEMM (starm_ttm_residual_bf16): the result
is fl(M @ x) of the reference to a few u, not merely the exact DCT.  Shorter
DCTs (n < 256: the dense DMMA product costs less than FFT + residual) and
any other matrix take the dense product.  STARM_EXACT_DCT=1 skips the
residual (diagnostic: the exact DCT-II alone).
"""

from __future__ import annotations

import os
from dataclasses import dataclass
from math import prod

import numpy as np

from . import _native as nat
from .tensors import DenseTensor, DeviceTensor, as_device
from .transform_set import DCT, IDENTITY, Transform, TransformSet

__all__ = ["BATCHED", "LOOP", "PARFOR", "VARIANTS", "TTMPlan", "ttm", "ttm_inverse",
           "to_transform_domain", "from_transform_domain", "ttm_device"]

BATCHED = "batched"
LOOP = "loop"
PARFOR = "parfor"
VARIANTS = (BATCHED, LOOP, PARFOR)


@dataclass(frozen=True)
class TTMPlan:
    """Geometry of one mode-k contraction (ttm.py:34-73)."""

    mode: int
    rows: int
    inner: int
    batch: int
    out_cols: int
    variant: str = BATCHED

    def __post_init__(self):
        if self.variant not in VARIANTS:
            raise ValueError(f"unknown ttm variant {self.variant!r}")

    @classmethod
    def for_dims(cls, dims, mode, out_cols, variant=BATCHED):
        dims = tuple(dims)
        mode = int(mode)
        if mode < 2:
            raise ValueError("the first two modes are never contracted")
        if mode >= len(dims):
            raise ValueError(f"mode {mode} out of range for {len(dims)} modes")
        return cls(mode, prod(dims[:mode]), dims[mode], prod(dims[mode + 1:]), int(out_cols), variant)

    @property
    def is_last_mode(self) -> bool:
        return self.batch == 1


def _threads(threads) -> int:
    threads = int(threads)
    if threads < 1:
        raise ValueError(f"thread count must be positive, got {threads}")
    return threads


def _matrix_operand(m, device, transpose=False):
    """Row-major device copy of M (or M^T) and its (out_cols, inner) shape."""
    import torch
    if isinstance(m, Transform):
        op = m.device_operand(device, transpose)
        return op, op.shape[0], op.shape[1]
    if isinstance(m, torch.Tensor):
        mat = m.to(device=device, dtype=torch.float64)
        if mat.dim() != 2:
            raise ValueError(f"expected a matrix, got {mat.dim()} modes")
        mat = (mat.T if transpose else mat).contiguous()
        return mat, mat.shape[0], mat.shape[1]
    mat = np.asarray(m, dtype=np.float64)
    if mat.ndim != 2:
        raise ValueError(f"expected a matrix, got {mat.ndim} modes")
    if transpose:
        mat = mat.T
    op = torch.from_numpy(np.ascontiguousarray(mat)).to(device)
    return op, mat.shape[0], mat.shape[1]


def ttm_device(x: DeviceTensor, mode: int, op, out_cols: int, inner: int) -> DeviceTensor:
    """One K1 launch: result.unfold(mode) = op @ x.unfold(mode)."""
    plan = TTMPlan.for_dims(x.dims, mode, out_cols)
    if inner != plan.inner:
        raise ValueError(f"matrix has {inner} columns, mode {plan.mode} extent is {plan.inner}")
    out_dims = x.dims[:mode] + (out_cols,) + x.dims[mode + 1:]
    out = DeviceTensor.empty(out_dims, x.device)
    nat.call("starm_ttm_f64", x.data.data_ptr(), op.data_ptr(), out.data.data_ptr(), plan.rows,
             plan.inner, plan.batch, out_cols, nat.stream_ptr(x.device))
    return out


DCT_FFT_MIN = 256   # below this the dense DMMA product is cheaper than FFT + residual


def _fast_kind(m, n):
    if isinstance(m, Transform):
        if (m.kind == DCT and DCT_FFT_MIN <= n <= 4096 and (n & (n - 1)) == 0
                and m.residual_host() is not None):
            return DCT
        if m.kind == IDENTITY:
            return IDENTITY
    return None


def structured_device(x: DeviceTensor, mode: int, kind: str, inverse: bool,
                      tr: Transform = None) -> DeviceTensor:
    """Mode-``mode`` product with a DCT (DCT-II, or DCT-III when inverse) or
    identity transform without the dense matrix.  For the DCT, ``tr``'s
    residual Delta = M - M_exact is added on the tensor cores so the result
    is the reference's dense product with tr.matrix (or its transpose)."""
    import torch
    plan = TTMPlan.for_dims(x.dims, mode, x.dims[mode])
    out = DeviceTensor.empty(x.dims, x.device)
    if kind == IDENTITY:
        out.data.copy_(x.data)
        return out
    st = nat.stream_ptr(x.device)
    if tr is None or os.environ.get("STARM_EXACT_DCT", "0") == "1":
        nat.call("starm_dct_f64", x.data.data_ptr(), out.data.data_ptr(), plan.rows, plan.inner,
                 plan.batch, int(bool(inverse)), st)
        return out
    op = tr.residual_operand(x.device, transpose=inverse)
    if op is None:
        raise ValueError("transform has no DCT residual operand")
    delta, e = op
    lib = nat.load()
    nbytes = lib.starm_ttm_residual_workspace_bytes(plan.rows, plan.inner, plan.batch)
    ws = torch.empty(nbytes + 128, dtype=torch.uint8, device=x.device)
    base = ws.data_ptr()
    base += (-base) % 128
    nat.call("starm_dct_residual_f64", x.data.data_ptr(), out.data.data_ptr(), plan.rows,
             plan.inner, plan.batch, int(bool(inverse)), delta.data_ptr(), int(e), base, nbytes, st)
    return out


def _shape(m):
    if isinstance(m, Transform):
        return m.matrix.shape
    if hasattr(m, "shape") and not isinstance(m, np.ndarray):
        return tuple(m.shape)
    return np.shape(m)


def _run(t, fn):
    """Host in -> host out; device in -> device out."""
    if isinstance(t, DeviceTensor):
        return fn(t)
    if not isinstance(t, DenseTensor):
        raise TypeError(f"expected DenseTensor or DeviceTensor, got {type(t).__name__}")
    dev = nat.require_cuda()
    return fn(as_device(t, dev)).to_host()


def ttm(t, mode, m, variant=BATCHED, threads=1):
    """Contract mode ``mode`` (>= 2) with ``m`` of shape (J, n_mode)."""
    _threads(threads)
    TTMPlan.for_dims(t.dims, mode, 1, variant)  # validates mode and variant
    shape = _shape(m)
    if len(shape) != 2:
        raise ValueError(f"expected a matrix, got {len(shape)} modes")
    if shape[1] != t.dims[mode]:
        raise ValueError(f"matrix has {shape[1]} columns, mode {mode} extent is {t.dims[mode]}")

    def go(x):
        kind = _fast_kind(m, x.dims[mode])
        if kind is not None:
            return structured_device(x, mode, kind, inverse=False, tr=m)
        op, j, n = _matrix_operand(m, x.device)
        return ttm_device(x, mode, op, j, n)

    return _run(t, go)


def ttm_inverse(t, mode, m, variant=BATCHED, threads=1):
    """Contract with m^T (ttm.py:107-110)."""
    _threads(threads)
    TTMPlan.for_dims(t.dims, mode, 1, variant)
    shape = _shape(m)
    if len(shape) != 2 or shape[0] != t.dims[mode]:
        raise ValueError(f"matrix of shape {shape} cannot undo mode {mode} of extent {t.dims[mode]}")

    def go(x):
        kind = _fast_kind(m, x.dims[mode])
        if kind is not None:
            return structured_device(x, mode, kind, inverse=True, tr=m)
        op, j, n = _matrix_operand(m, x.device, transpose=True)
        return ttm_device(x, mode, op, j, n)

    return _run(t, go)


def forward_device(x: DeviceTensor, ts: TransformSet) -> DeviceTensor:
    out = x
    for k, tr in enumerate(ts, start=2):
        kind = _fast_kind(tr, out.dims[k])
        if kind is not None:
            out = structured_device(out, k, kind, inverse=False, tr=tr)
            continue
        op, j, n = _matrix_operand(tr, x.device)
        out = ttm_device(out, k, op, j, n)
    return out


def inverse_device(x: DeviceTensor, ts: TransformSet) -> DeviceTensor:
    out = x
    for k in range(len(ts) + 1, 1, -1):
        kind = _fast_kind(ts[k - 2], out.dims[k])
        if kind is not None:
            out = structured_device(out, k, kind, inverse=True, tr=ts[k - 2])
            continue
        op, j, n = _matrix_operand(ts[k - 2], x.device, transpose=True)
        out = ttm_device(out, k, op, j, n)
    return out


def to_transform_domain(t, ts: TransformSet, variant=BATCHED, threads=1):
    """Ascending modes (ttm.py:138-144)."""
    _threads(threads)
    if variant not in VARIANTS:
        raise ValueError(f"unknown ttm variant {variant!r}")
    ts.check_dims(t.dims)
    return _run(t, lambda x: forward_device(x, ts))


def from_transform_domain(t, ts: TransformSet, variant=BATCHED, threads=1):
    """Descending modes with the transposes (ttm.py:147-153)."""
    _threads(threads)
    if variant not in VARIANTS:
        raise ValueError(f"unknown ttm variant {variant!r}")
    ts.check_dims(t.dims)
    return _run(t, lambda x: inverse_device(x, ts))


PIPELINE_BLOCKS = 16            # fibre runs of the pipelined host upload
PIPELINE_MIN_BYTES = 64 << 20   # smaller tensors upload in one piece
_COPY_STREAMS = {}


def _copy_stream(dev):
    import torch
    idx = dev.index if dev.index is not None else torch.cuda.current_device()
    if idx not in _COPY_STREAMS:
        _COPY_STREAMS[idx] = torch.cuda.Stream(torch.device("cuda", idx))
    return _COPY_STREAMS[idx]


def pipelined_upload_applies(a, ts: TransformSet) -> bool:
    """True for a host tensor whose forward transform is the deferrable DCT
    and which is large enough for the block-wise upload to pay."""
    return (isinstance(a, DenseTensor) and os.environ.get("STARM_PIPELINE", "1") != "0"
            and deferrable(ts, a.dims) and a.data.nbytes >= PIPELINE_MIN_BYTES)


def forward_from_host(a: DenseTensor, ts: TransformSet, dev):
    """Forward transform of a HOST 3-way tensor whose single transform takes
    the dense DMMA product, block by block: the strided host-to-device copy of
    fibre run g+1 (starm_copy2d_h2d, copy stream) overlaps the product of run
    g (starm_ttm_block_f64); the result is bitwise forward_device's (every
    output element is the same dot product in the same order).  Returns None
    when it does not apply (other shapes / kinds, small tensors): the caller
    uploads in one piece."""
    import torch
    if (not isinstance(a, DenseTensor) or os.environ.get("STARM_PIPELINE", "1") == "0"
            or len(a.dims) != 3 or len(ts) != 1 or a.data.nbytes < PIPELINE_MIN_BYTES
            or _fast_kind(ts[0], a.dims[2]) is not None):
        return None
    m, p, n = a.dims
    rows = m * p
    op, j, inner = _matrix_operand(ts[0], dev)
    if j != n or inner != n:
        return None
    host = a.data
    if host.dtype != np.float64 or not host.flags.c_contiguous:
        return None
    out = DeviceTensor.empty(a.dims, dev)
    x = torch.empty(rows * n, dtype=torch.float64, device=dev)
    step = max(128, -(-rows // PIPELINE_BLOCKS + 127) // 128 * 128)
    compute = torch.cuda.current_stream(dev)
    copy = _copy_stream(dev)
    copy.wait_stream(compute)
    x.record_stream(copy)
    hc, hs = nat.register_stream(copy), nat.stream_ptr(dev)
    src0 = host.ctypes.data
    for f0 in range(0, rows, step):
        nf = min(step, rows - f0)
        nat.call("starm_copy2d_h2d", x.data_ptr() + 8 * f0, 8 * rows, src0 + 8 * f0, 8 * rows,
                 8 * nf, n, hc)
        ev = torch.cuda.Event()
        ev.record(copy)
        compute.wait_event(ev)
        nat.call("starm_ttm_block_f64", x.data_ptr(), op.data_ptr(), out.data.data_ptr(), rows, n, n,
                 f0, nf, hs)
    return out


def upload_forward(a, ts: TransformSet, dev) -> DeviceTensor:
    """Transform-domain tensor (device) of a host or device tensor: host
    tensors that qualify go through the block-wise upload."""
    if isinstance(a, DenseTensor):
        out = forward_from_host(a, ts, dev)
        if out is not None:
            return out
    return forward_device(as_device(a, dev), ts)


class DeferredResidual:
    """The exact FFT DCT of a tensor whose reference-operator residual
    (starm_ttm_residual_bf16) has NOT been added yet: the bf16 operand is
    kept in ``ws`` so the residual can be applied later to all output slices
    (``apply_all``) or only to a selection of them (``apply_cols`` on a
    gathered copy): the pruned tolerance path corrects only the slices it
    keeps.  3-way tensors, forward DCT-II, n in [256, 4096]."""

    def __init__(self, x: DeviceTensor, tr: Transform):
        import torch
        m, p, n = x.dims
        self.tr, self.rows, self.n, self.device = tr, m * p, n, x.device
        lib = nat.load()
        nbytes = lib.starm_ttm_residual_workspace_bytes(self.rows, n, 1)
        self._ws = torch.empty(nbytes + 128, dtype=torch.uint8, device=x.device)
        self.base = self._ws.data_ptr() + (-self._ws.data_ptr()) % 128
        self.out = DeviceTensor.empty(x.dims, x.device)
        self.energies = None
        nat.call("starm_dct_pack_f64", x.data.data_ptr(), self.out.data.data_ptr(), self.rows, n, 1,
                 0, self.base, nbytes, nat.stream_ptr(x.device))

    @classmethod
    def from_host(cls, a: DenseTensor, tr: Transform, dev, blocks=None):
        """The same state for a HOST tensor, built block by block: the m*p
        fibres are cut into ``blocks`` runs (multiples of 128 fibres); the
        strided host-to-device copy of run g+1 (starm_copy2d_h2d on a copy
        stream) overlaps the FFT DCT, the bf16 operand rows and the partial
        slice energies of run g (starm_dct_pack_block_f64,
        starm_slice_energy_block_f64), so that when the last bytes have
        crossed PCIe the transform-domain tensor and its slice energies
        (``self.energies``, device, summed over the runs in order) are nearly
        complete.  Every fibre goes through the same kernel as in __init__, so
        ``out`` and the operand are bit-identical to the one-shot path."""
        import torch
        m, p, n = a.dims
        rows = m * p
        self = cls.__new__(cls)
        self.tr, self.rows, self.n, self.device = tr, rows, n, dev
        lib = nat.load()
        nbytes = lib.starm_ttm_residual_workspace_bytes(rows, n, 1)
        self._ws = torch.empty(nbytes + 128, dtype=torch.uint8, device=dev)
        self.base = self._ws.data_ptr() + (-self._ws.data_ptr()) % 128
        self.out = DeviceTensor.empty(a.dims, dev)
        host = a.data
        if not (host.flags.f_contiguous or host.flags.c_contiguous) or host.dtype != np.float64:
            host = np.ascontiguousarray(host.reshape(-1, order="F"))
        nb = int(blocks or PIPELINE_BLOCKS)
        step = max(128, -(-rows // nb + 127) // 128 * 128)
        starts = list(range(0, rows, step))
        x = torch.empty(rows * n, dtype=torch.float64, device=dev)
        parts = torch.empty((len(starts), n), dtype=torch.float64, device=dev)
        compute = torch.cuda.current_stream(dev)
        copy = _copy_stream(dev)
        copy.wait_stream(compute)       # x may reuse a block with compute work pending
        x.record_stream(copy)
        hc, hs = nat.register_stream(copy), nat.stream_ptr(dev)
        src0 = host.ctypes.data
        for g, f0 in enumerate(starts):
            nf = min(step, rows - f0)
            nat.call("starm_copy2d_h2d", x.data_ptr() + 8 * f0, 8 * rows, src0 + 8 * f0, 8 * rows,
                     8 * nf, n, hc)
            ev = torch.cuda.Event()
            ev.record(copy)
            compute.wait_event(ev)
            nat.call("starm_dct_pack_block_f64", x.data_ptr(), self.out.data.data_ptr(), rows, n,
                     f0, nf, self.base, nbytes, hs)
            nat.call("starm_slice_energy_block_f64", self.out.data.data_ptr(), rows, n, f0, nf,
                     parts[g].data_ptr(), hs)
        self.energies = parts.sum(dim=0) if len(starts) > 1 else parts[0]
        self._keep = (host, x)          # alive until the queued work has consumed them
        return self

    def _apply(self, dst, delta_rows, nout):
        op = self.tr.residual_operand(self.device)
        delta, e = op
        nat.call("starm_residual_apply_f64", self.base, delta_rows.data_ptr(), int(e),
                 dst.data_ptr(), self.rows, self.n, nout, 1, nat.stream_ptr(self.device))

    def apply_all(self, dst=None):
        """Complete the reference operator on every slice of ``self.out``."""
        delta, _ = self.tr.residual_operand(self.device)
        self._apply((dst if dst is not None else self.out.data), delta, self.n)

    def apply_cols(self, sub, ids_dev):
        """``sub`` (rows x len(ids)) holds FFT-only slices ``ids`` of out: add
        their residual columns (Delta rows ids, zero-padded to 256)."""
        import torch
        delta, _ = self.tr.residual_operand(self.device)
        ns = int(ids_dev.numel())
        pad = ((ns + 255) // 256) * 256
        sel = torch.zeros((pad, self.n), dtype=delta.dtype, device=self.device)
        sel[:ns] = delta.view(self.n, self.n).index_select(0, ids_dev)
        self._apply(sub, sel, ns)


def deferrable(ts: TransformSet, dims) -> bool:
    """True when the forward transform is one DCT-kind mode with the FFT +
    residual route (so the residual can be deferred)."""
    if len(dims) != 3 or len(ts) != 1 or os.environ.get("STARM_EXACT_DCT", "0") == "1":
        return False
    return _fast_kind(ts[0], dims[2]) == DCT

