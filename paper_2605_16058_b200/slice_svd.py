"""Slice-wise thin SVDs on the B200 (reference slicesvd.py).

All factorizations run in the batched slice-SVD kernels (csrc/svd_f64.cu)
through ``starm_svd_f64``: Householder QR + band reduction + bulge chasing
+ bisection/Laguerre for sigma, inverse iteration + back-transformation for
vectors, and a blocked one-sided Jacobi kernel for slices too tall for the
shared-memory panel.  The reference's two threading strategies
(``slices-parallel`` / ``svd-parallel``, slicesvd.py:65-77) are validated
and then map to the same persistent grids.  Inputs are never modified: the
kernels factor a private workspace copy of each slice.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _native as nat
from .tensors import DenseTensor, DeviceTensor, as_device, device_to_host

__all__ = ["SLICES_PARALLEL", "SVD_PARALLEL", "STRATEGIES", "SliceSVDSet", "VariableRankFactors",
           "DeviceFactors", "svd_all_slices", "svd_values_only", "svd_truncated_slices",
           "svd_values_device", "svd_truncated_device", "svd_full_device"]

SLICES_PARALLEL = "slices-parallel"
SVD_PARALLEL = "svd-parallel"
STRATEGIES = (SLICES_PARALLEL, SVD_PARALLEL)

def _check_strategy(strategy, threads):
    if strategy not in STRATEGIES:
        raise ValueError(f"unknown slice SVD strategy {strategy!r}")
    threads = int(threads)
    if threads < 1:
        raise ValueError(f"thread count must be positive, got {threads}")


def _geometry(t):
    if len(t.dims) < 3:
        raise ValueError("slicewise SVD applies to tensors with at least three modes")
    m, p = t.dims[0], t.dims[1]
    return m, p, min(m, p), t.num_slices


@dataclass(eq=False)
class SliceSVDSet:
    """u (m, r, N), s (r, N) descending per column, v (p, r, N) (slicesvd.py:87-112).
    Host inputs give DenseTensor/ndarray fields, device inputs give
    DeviceTensor/torch fields."""

    u: object
    s: object
    v: object

    @property
    def rank(self) -> int:
        return self.s.shape[0]

    @property
    def num_slices(self) -> int:
        return self.s.shape[1]

    def reconstruct_slice(self, i) -> np.ndarray:
        i = int(i)
        u = self.u if isinstance(self.u, DenseTensor) else self.u.to_host()
        v = self.v if isinstance(self.v, DenseTensor) else self.v.to_host()
        s = np.asarray(self.s if isinstance(self.s, np.ndarray) else self.s.cpu().numpy())
        return u.frontal_slice(i) @ (s[:, i, None] * v.frontal_slice(i).T)


class VariableRankFactors:
    """Packed, unpadded leading triplets (slicesvd.py:180-256): slice i owns
    an (m x ranks[i]) column-major block of ``u_data`` and a (ranks[i] x p)
    block of diag(s) V^T in ``g_data``, concatenated in slice order."""

    def __init__(self, slice_rows, slice_cols, ranks, u_data, g_data):
        self.slice_rows = int(slice_rows)
        self.slice_cols = int(slice_cols)
        ranks = np.asarray(ranks, dtype=np.int64)
        if ranks.ndim != 1:
            raise ValueError("ranks must be a flat sequence")
        bound = min(self.slice_rows, self.slice_cols)
        if ranks.size and (ranks.min() < 0 or ranks.max() > bound):
            raise ValueError(f"ranks must lie in [0, {bound}]")
        self.ranks = ranks
        self.u_data = np.ascontiguousarray(u_data, dtype=np.float64).reshape(-1)
        self.g_data = np.ascontiguousarray(g_data, dtype=np.float64).reshape(-1)
        self._u_offsets = np.concatenate([[0], np.cumsum(ranks * self.slice_rows)]).astype(np.int64)
        self._g_offsets = np.concatenate([[0], np.cumsum(ranks * self.slice_cols)]).astype(np.int64)
        if self.u_data.size != self._u_offsets[-1]:
            raise ValueError(f"left-vector payload holds {self.u_data.size} values, "
                             f"ranks call for {int(self._u_offsets[-1])}")
        if self.g_data.size != self._g_offsets[-1]:
            raise ValueError(f"product payload holds {self.g_data.size} values, "
                             f"ranks call for {int(self._g_offsets[-1])}")

    @classmethod
    def allocate(cls, slice_rows, slice_cols, ranks):
        ranks = np.asarray(ranks, dtype=np.int64)
        return cls(slice_rows, slice_cols, ranks, np.empty(int((ranks * slice_rows).sum())),
                   np.empty(int((ranks * slice_cols).sum())))

    @property
    def num_slices(self) -> int:
        return self.ranks.size

    @property
    def total_rank(self) -> int:
        return int(self.ranks.sum())

    def u_block(self, i) -> np.ndarray:
        a, b = self._u_offsets[i], self._u_offsets[i + 1]
        return self.u_data[a:b].reshape((self.slice_rows, int(self.ranks[i])), order="F")

    def g_block(self, i) -> np.ndarray:
        a, b = self._g_offsets[i], self._g_offsets[i + 1]
        return self.g_data[a:b].reshape((int(self.ranks[i]), self.slice_cols), order="F")

    def to_host(self) -> "VariableRankFactors":
        return self


class DeviceFactors:
    """HBM twin of VariableRankFactors: ranks / offsets / payloads as torch
    CUDA tensors (offsets have N+1 entries).  ``total_rank`` is host-known."""

    def __init__(self, slice_rows, slice_cols, ranks, u_off, g_off, u_data, g_data, total_rank):
        self.slice_rows = int(slice_rows)
        self.slice_cols = int(slice_cols)
        self.ranks_dev = ranks
        self.u_off = u_off
        self.g_off = g_off
        self.u_data = u_data
        self.g_data = g_data
        self.total_rank = int(total_rank)
        self._host_ranks = None

    @property
    def num_slices(self) -> int:
        return int(self.ranks_dev.numel())

    @property
    def ranks(self) -> np.ndarray:
        if self._host_ranks is None:
            self._host_ranks = self.ranks_dev.cpu().numpy().astype(np.int64)
        return self._host_ranks

    def to_host(self) -> VariableRankFactors:
        u, g = device_to_host(self.u_data, self.g_data)
        return VariableRankFactors(self.slice_rows, self.slice_cols, self.ranks, u, g)


# ---------------------------------------------------------------- launches

def _raise_slice_status(status_host, what):
    bad, noconv = int(status_host[0]), int(status_host[1])
    if bad != 2**31 - 1:
        raise ValueError(f"slice {bad} contains non-finite values")
    if noconv != 2**31 - 1:
        raise np.linalg.LinAlgError(f"SVD did not converge on slice {noconv} ({what})")


def _svd_launch(x: DeviceTensor, job, ids=None, s=None, u=None, v=None, ranks=None, u_off=None,
                g_off=None, u_data=None, g_data=None, ws=None, defer=None):
    """One call of starm_svd_f64 over ``ids`` (device int64, or None for every
    slice).  Returns the workspace (which carries the per-slice state after a
    VALUES_STATE job).  Work is scheduled on persistent grids; the scratch is
    per resident CTA except for the per-slice factorisation state.  With a
    ``defer`` list the device status pair is appended to it instead of being
    read back here (the caller checks it with ``check_status`` at its next
    synchronisation point, before any result is returned)."""
    import torch
    m, p, r, n = _geometry(x)
    dev = x.device
    count = n if ids is None else int(ids.numel())
    if count == 0:
        return ws
    status = torch.empty(2, dtype=torch.int32, device=dev)
    lib = nat.load()
    nbytes = lib.starm_svd_workspace_bytes(m, p, n, count, job)
    if ws is None:
        ws = nat.workspace(nbytes, dev)
    elif ws.numel() < nbytes:
        raise RuntimeError(f"SVD state workspace too small ({ws.numel()} < {nbytes} bytes)")
    nat.call("starm_svd_f64", x.data.data_ptr(), m, p, n, nat.ptr(ids), count, job, nat.ptr(s),
             nat.ptr(u), nat.ptr(v), nat.ptr(ranks), nat.ptr(u_off), nat.ptr(g_off),
             nat.ptr(u_data), nat.ptr(g_data), status.data_ptr(), ws.data_ptr(), ws.numel(),
             nat.stream_ptr(dev))
    if defer is not None:
        defer.append(status)
    else:
        _raise_slice_status(status.cpu().numpy(), "slice SVD")
    return ws


def check_status(statuses_host):
    """Raise for the first failing deferred status pair (host int values)."""
    for i in range(0, len(statuses_host), 2):
        _raise_slice_status(statuses_host[i:i + 2], "slice SVD")


class SvdState:
    """Factorisation state of every slice kept in HBM by a VALUES_STATE pass
    (bidiagonals and logged right-side transformations); lets the truncated
    pass skip refactoring (the device form of the compute-efficient strategy)."""

    def __init__(self, ws, s):
        self.ws = ws
        self.s = s


def state_bytes(x: DeviceTensor) -> int:
    m, p, r, n = _geometry(x)
    return int(nat.load().starm_svd_workspace_bytes(m, p, n, n, nat.SVD_VALUES_STATE))


def svd_values_device(x: DeviceTensor, keep_state=False, defer=None):
    """(r, N) singular values as a column-major torch tensor (flat r*N); with
    ``keep_state`` also returns the SvdState for svd_truncated_device."""
    import torch
    m, p, r, n = _geometry(x)
    s = torch.empty(r * n, dtype=torch.float64, device=x.device)
    if keep_state:
        lib = nat.load()
        if (lib.starm_svd_workspace_bytes(m, p, n, n, nat.SVD_VALUES_STATE)
                == lib.starm_svd_workspace_bytes(m, p, n, n, nat.SVD_VALUES)):
            # slices outside the bidiagonal path (Jacobi kernel) keep no
            # state: the truncated pass refactors them
            _svd_launch(x, nat.SVD_VALUES, s=s, defer=defer)
            return s, None
        ws = _svd_launch(x, nat.SVD_VALUES_STATE, s=s, defer=defer)
        return s, SvdState(ws, s)
    _svd_launch(x, nat.SVD_VALUES, s=s, defer=defer)
    return s


def svd_full_device(x: DeviceTensor):
    import torch
    m, p, r, n = _geometry(x)
    s = torch.empty(r * n, dtype=torch.float64, device=x.device)
    u = torch.empty(m * r * n, dtype=torch.float64, device=x.device)
    v = torch.empty(p * r * n, dtype=torch.float64, device=x.device)
    _svd_launch(x, nat.SVD_FULL, s=s, u=u, v=v)
    return s, u, v


def pack_offsets_device(ranks_dev, m, p):
    import torch
    n = int(ranks_dev.numel())
    u_off = torch.empty(n + 1, dtype=torch.int64, device=ranks_dev.device)
    g_off = torch.empty(n + 1, dtype=torch.int64, device=ranks_dev.device)
    nat.call("starm_pack_offsets", ranks_dev.data_ptr(), n, m, p, u_off.data_ptr(),
             g_off.data_ptr(), nat.stream_ptr(ranks_dev.device))
    return u_off, g_off


def svd_truncated_device(x: DeviceTensor, ranks_dev, total_rank, ids=None, keep_values=False,
                         state=None, defer=None):
    """Packed leading-rank factors.  ``ids`` lists the slices to factor
    (device int64); by default all slices with rank > 0, or every slice
    when ``keep_values``.  With ``state`` (from svd_values_device(...,
    keep_state=True)) the slices are not refactored.  Returns
    (DeviceFactors, s or None)."""
    import torch
    m, p, r, n = _geometry(x)
    dev = x.device
    u_off, g_off = pack_offsets_device(ranks_dev, m, p)
    u_data = torch.empty(max(total_rank * m, 1), dtype=torch.float64, device=dev)
    g_data = torch.empty(max(total_rank * p, 1), dtype=torch.float64, device=dev)
    s = torch.empty(r * n, dtype=torch.float64, device=dev) if keep_values else None
    if state is not None and not keep_values:
        pass  # the state pass walks every slice by index and skips rank-0 ones (no host sync)
    elif not keep_values and ids is None:
        ids = torch.nonzero(ranks_dev > 0).reshape(-1).to(torch.int64)
    if keep_values:
        ids = None
    if ids is None or ids.numel() > 0:
        if state is not None and not keep_values:
            _svd_launch(x, nat.SVD_TRUNCATED_STATE, ids=ids, s=state.s, ranks=ranks_dev,
                        u_off=u_off, g_off=g_off, u_data=u_data, g_data=g_data, ws=state.ws,
                        defer=defer)
        else:
            _svd_launch(x, nat.SVD_TRUNCATED, ids=ids, s=s, ranks=ranks_dev, u_off=u_off,
                        g_off=g_off, u_data=u_data, g_data=g_data, defer=defer)
    factors = DeviceFactors(m, p, ranks_dev, u_off, g_off, u_data[: total_rank * m],
                            g_data[: total_rank * p], total_rank)
    return factors, s


# ------------------------------------------------------------ public API

def svd_all_slices(ahat, strategy=SLICES_PARALLEL, threads=1) -> SliceSVDSet:
    """Every slice's thin SVD (slicesvd.py:115-136)."""
    _check_strategy(strategy, threads)
    m, p, r, n = _geometry(ahat)
    host = isinstance(ahat, DenseTensor)
    x = as_device(ahat, nat.require_cuda() if host else None)
    s, u, v = svd_full_device(x)
    if host:
        return SliceSVDSet(DenseTensor(u.cpu().numpy(), (m, r, n), copy=False),
                           s.cpu().numpy().reshape((r, n), order="F"),
                           DenseTensor(v.cpu().numpy(), (p, r, n), copy=False))
    return SliceSVDSet(DeviceTensor(u, (m, r, n)), s.reshape(n, r).T, DeviceTensor(v, (p, r, n)))


def svd_values_only(ahat, strategy=SLICES_PARALLEL, threads=1):
    """(r, N) singular values; bitwise equal to svd_all_slices' s
    (slicesvd.py:171-177) because both jobs run the same rotation sequence."""
    _check_strategy(strategy, threads)
    m, p, r, n = _geometry(ahat)
    host = isinstance(ahat, DenseTensor)
    x = as_device(ahat, nat.require_cuda() if host else None)
    s = svd_values_device(x)
    if host:
        return s.cpu().numpy().reshape((r, n), order="F")
    return s.reshape(n, r).T


def svd_truncated_slices(ahat, ranks, strategy=SLICES_PARALLEL, threads=1, keep_values=False):
    """Leading-rank packed factors (slicesvd.py:259-292)."""
    import torch
    _check_strategy(strategy, threads)
    m, p, r, n = _geometry(ahat)
    if isinstance(ranks, torch.Tensor):  # e.g. ThresholdResult.ranks of a device compute_threshold
        ranks = ranks.cpu().numpy()
    ranks = np.asarray(ranks, dtype=np.int64)
    if ranks.shape != (n,):
        raise ValueError(f"need one rank per slice ({n}), got shape {ranks.shape}")
    if ranks.size and (ranks.min() < 0 or ranks.max() > r):
        raise ValueError(f"ranks must lie in [0, {r}]")
    host = isinstance(ahat, DenseTensor)
    x = as_device(ahat, nat.require_cuda() if host else None)
    ranks_dev = torch.from_numpy(ranks).to(x.device)
    ids = None
    if not keep_values:
        nz = np.flatnonzero(ranks > 0).astype(np.int64)
        ids = torch.from_numpy(nz).to(x.device)
    factors, s = svd_truncated_device(x, ranks_dev, int(ranks.sum()), ids=ids,
                                      keep_values=keep_values)
    factors._host_ranks = ranks
    if host:
        f = factors.to_host()
        if keep_values:
            return f, s.cpu().numpy().reshape((r, n), order="F")
        return f
    if keep_values:
        return factors, s.reshape(n, r).T
    return factors
