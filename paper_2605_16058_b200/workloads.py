"""The BASELINE.json configurations as runnable workloads (bench.py, scripts).

Each workload builds its seeded synthetic input (configs.py), holds it in
HBM, and runs ONE compression call through the public API per ``step``:

  c1   256 x 256 x 64 f64, DCT-II (n = 64: dense DMMA product), fixed rank 10
  c2   361 x 720 x 1024 f64, DCT-II (FFT + tcgen05 residual), tolerance 1e-2
  c3   1024 x 1024 x 512 f64, Haar M (dense DMMA product), fixed rank 32
  c4   512 x 512 x 2048 f32 frames upcast to f64 (tensor.py:87), raw
       M = I + 0.1 N/sqrt(n) (ttm.py:76-77 accepts it), tolerance 1e-3:
       SURVEY 8c's restatement (values -> threshold -> truncated), error with
       the explicit M^-1
  c5   8192 x 64 x 4096 f64, Haar M, fixed rank 16   (A = Ahat x3 M^T formed
  c5t  the same tensor, tolerance 1e-4                 on the device)

``flops`` gives the algorithmic work of BASELINE.md section 3 (the GVL
necessary-output count for the SVD, 2 n^2 m p per transform) so bench.py can
state roofline fractions.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from . import configs as cf

__all__ = ["WORKLOADS", "Workload", "make_workload"]


@dataclass
class Workload:
    name: str
    dims: tuple
    kind: str                 # "fixed-rank" | "tolerance"
    param: float              # rank or epsilon
    transform: str            # "dct" | "haar" | "raw"
    describe: str
    host: object = None       # F-order float64 host array (None when formed on the device)
    ts: object = None
    mat: object = None        # raw M (c4)
    minv: object = None       # explicit M^-1 (c4)
    extra: dict = field(default_factory=dict)

    @property
    def in_bytes(self) -> int:
        """Input bytes of one call: float32 frames for c4, else f64."""
        item = 4 if (self.host is not None and self.host.dtype == np.float32) else 8
        return int(np.prod(self.dims)) * item

    # ------------------------------------------------------------ device
    def device_input(self, dev):
        """The input tensor resident in HBM (DeviceTensor)."""
        import paper_2605_16058_b200 as sb
        if self.host is not None and self.host.dtype == np.float32:
            return sb.DeviceTensor.from_host(self.host, dev)   # f32 H2D + device upcast
        if self.host is not None:
            return sb.DeviceTensor.from_host(sb.DenseTensor(self.host, copy=False), dev)
        ahat = self.extra["ahat"]
        from .mode_product import inverse_device
        xh = sb.DeviceTensor.from_host(sb.DenseTensor(ahat, copy=False), dev)
        return inverse_device(xh, self.ts)       # A = Ahat x3 M^T

    def step(self, x, clock=None):
        """One compression call on a DeviceTensor; returns a result exposing
        ``factors``, ``discarded_energy``, ``total_energy``."""
        import paper_2605_16058_b200 as sb
        if self.transform == "raw":
            return _c4_step(x, self.mat, self.param, clock)
        if self.kind == "fixed-rank":
            return sb.tsvdm_fixed_rank(x, self.ts, int(self.param))
        return sb.tsvdm_tolerance(x, self.ts, float(self.param), clock=clock)

    def forward(self, x):
        """The forward transform alone (for the roofline split)."""
        import paper_2605_16058_b200 as sb
        if self.transform == "raw":
            return sb.ttm(x, 2, self.mat)
        from .mode_product import forward_device
        return forward_device(x, self.ts)

    def realised_error(self, x, res):
        """(realised relative error, recorded sqrt(disc/total)) of a step
        result, through the device reconstruction and the K10 error kernel.
        c4 reports the transform-domain error (M is not orthonormal; the
        original-domain error is in ``extra['orig_error']``)."""
        import paper_2605_16058_b200 as sb
        from .compress import reconstruct_device, relative_error_device
        recorded = math.sqrt(res.discarded_energy / res.total_energy) if res.total_energy else 0.0
        if self.transform == "raw":
            chat = _unpack(res.factors, x.dims, x.device)
            ahat = self.forward(x)
            err_t = relative_error_device(ahat, chat)
            rec = sb.ttm(chat, 2, self.minv)
            self.extra["orig_error"] = relative_error_device(x, rec)
            return err_t, recorded
        if len(self.dims) == 3:
            from .compress import CompressedTensor, reconstruct_fused
            c = CompressedTensor(self.dims, self.ts, res.factors, "tsvdm1", 1.0) \
                if not isinstance(res, CompressedTensor) else res
            _, err = reconstruct_fused(c, a=x)   # K9 + inverse transform + K10 in one call
            return err, recorded
        rec = reconstruct_device(res, x.device)
        return relative_error_device(x, rec), recorded

    def flops(self, total_rank):
        """(transform flops one direction, SVD necessary flops, LAPACK-equiv)."""
        m, p, n = self.dims
        a, b = max(m, p), min(m, p)
        f_ttm = 2.0 * n * n * m * p
        f_sig = 2 * a * b * b + 2 * b ** 3
        f_uv = 6 * a * b * b + 20 * b ** 3
        f_svd = n * f_sig + (total_rank / b) * (f_uv - f_sig)
        return f_ttm, f_svd, n * f_uv


class _C4Result:
    def __init__(self, factors, thr):
        self.factors = factors
        self.discarded_energy = thr[1]
        self.total_energy = thr[2]
        self.tau = thr[0]


def _c4_step(x, mat, eps, clock=None):
    """SURVEY 8c config-4 restatement on the device: Ahat = ttm(A, 2, M) with
    the raw matrix, values pass keeping each slice's state, device threshold,
    truncated factors from the state (tsvdm_tolerance's schedule)."""
    import paper_2605_16058_b200 as sb
    from .compress import _summary, threshold_device
    from .slice_svd import svd_truncated_device, svd_values_device
    ahat = sb.ttm(x, 2, mat)
    s, state = svd_values_device(ahat, keep_state=True)
    m, p, n = ahat.dims
    ranks, scal, _, _, _ = threshold_device(s, min(m, p), n, eps)
    tau, disc, tot, total_rank = _summary(ranks, scal)
    f, _ = svd_truncated_device(ahat, ranks, total_rank, state=state)
    del state
    return _C4Result(f, (tau, disc, tot))


def _unpack(f, dims, dev):
    import paper_2605_16058_b200 as sb
    from . import _native as nat
    m, p, n = dims
    chat = sb.DeviceTensor.empty(dims, dev)
    nat.call("starm_unpack_facewise_f64", f.u_data.data_ptr(), f.g_data.data_ptr(),
             f.ranks_dev.data_ptr(), f.u_off.data_ptr(), f.g_off.data_ptr(), m, p, n,
             chat.data.data_ptr(), nat.stream_ptr(dev))
    return chat


WORKLOADS = ("c1", "c2", "c3", "c4", "c5", "c5t")


def make_workload(name, seed=0, scale=None):
    """Build workload ``name``.  ``scale`` (tests only) shrinks the extents."""
    import paper_2605_16058_b200 as sb
    if name == "c1":
        a = cf.config1(seed=seed)
        return Workload("c1", a.shape, "fixed-rank", 10, "dct",
                        "c1: 256x256x64 f64 rank-10 + 1e-3 noise, DCT-II, fixed rank 10",
                        host=a, ts=sb.TransformSet.build(a.shape, "dct"))
    if name == "c2":
        kw = dict(nlat=361, nlon=720, nt=1024) if scale is None else scale
        a = cf.config2(seed=seed, **kw)
        return Workload("c2", a.shape, "tolerance", 1e-2, "dct",
                        "c2: 361x720x1024 f64 climate-like, DCT-II over time, tolerance 1e-2, "
                        "memory-efficient", host=a, ts=sb.TransformSet.build(a.shape, "dct"))
    if name == "c3":
        kw = {} if scale is None else scale
        a, mm = cf.config3(seed=seed, **kw)
        return Workload("c3", a.shape, "fixed-rank", 32 if scale is None else 8, "haar",
                        "c3: 1024x1024x512 f64 CFD-like traveling modes, Haar M, fixed rank 32",
                        host=a, ts=sb.TransformSet((sb.validate_transform(mm),)))
    if name == "c4":
        kw = {} if scale is None else scale
        a32, mm, minv = cf.config4(seed=seed, **kw)
        # float32 frames stay float32 on the host; the tensor.py:87 upcast runs
        # on the device after the (half-size) H2D
        return Workload("c4", a32.shape, "tolerance", 1e-3, "raw",
                        "c4: 512x512x2048 X-ray-like f32 frames (upcast to f64 on the device), "
                        "raw invertible M = I + 0.1 N/sqrt(n), tolerance 1e-3, explicit M^-1",
                        host=np.asfortranarray(a32), mat=mm, minv=minv)
    if name in ("c5", "c5t"):
        kw = {} if scale is None else scale
        ahat, mm = cf.config5_transform_domain(seed=seed, **kw)
        ts = sb.TransformSet((sb.validate_transform(mm),))
        kind, param = ("fixed-rank", 16) if name == "c5" else ("tolerance", 1e-4)
        what = "fixed rank 16" if name == "c5" else "tolerance 1e-4"
        return Workload(name, ahat.shape, kind, param, "haar",
                        f"c5: 8192x64x4096 f64, sigma_j = 0.8^j per slice, Haar U/V/M, {what}",
                        ts=ts, extra={"ahat": ahat, "mat": mm})
    raise ValueError(f"unknown workload {name!r} (choose from {WORKLOADS})")
