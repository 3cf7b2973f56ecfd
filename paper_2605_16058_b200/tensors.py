"""Tensor carriers: the host ``DenseTensor`` of the reference API and its
device-resident twin ``DeviceTensor``.

``DenseTensor`` keeps the reference contract (tensor.py:76-173): float64,
column-major, read-only after construction, frontal slice i is the
contiguous m*p block at offset i*m*p.  ``DeviceTensor`` holds the same flat
column-major float64 buffer in HBM (a 1-D torch CUDA tensor), so a slice
is still a contiguous block and every kernel reads it in place.
"""

from __future__ import annotations

from dataclasses import dataclass
from math import prod

import os

import numpy as np

__all__ = ["linear_index", "multi_index", "SliceIndex", "DenseTensor", "DeviceTensor", "refold",
           "as_device", "is_device"]


def linear_index(dims, idx) -> int:
    """Column-major offset, first mode fastest (tensor.py:11-38)."""
    dims = tuple(dims)
    if len(idx) != len(dims):
        raise ValueError(f"index has {len(idx)} modes, tensor has {len(dims)}")
    off, stride = 0, 1
    for mode, (i, n) in enumerate(zip(idx, dims)):
        if i < 0 or i >= n:
            raise IndexError(f"index {i} out of range [0, {n}) in mode {mode}")
        off += int(i) * stride
        stride *= int(n)
    return off


def multi_index(dims, offset) -> tuple:
    """Inverse of linear_index (tensor.py:41-49)."""
    dims = tuple(dims)
    total = prod(dims)
    if offset < 0 or offset >= total:
        raise IndexError(f"offset {offset} out of range [0, {total})")
    out = []
    rem = int(offset)
    for n in dims:
        rem, r = divmod(rem, n)
        out.append(r)
    return tuple(out)


@dataclass(frozen=True)
class SliceIndex:
    """Frontal-slice address: trailing indices and the flat slice number."""

    trailing: tuple
    flat: int

    @classmethod
    def from_trailing(cls, dims, trailing):
        tr = tuple(int(i) for i in trailing)
        return cls(tr, linear_index(tuple(dims)[2:], tr))

    @classmethod
    def from_flat(cls, dims, flat):
        return cls(multi_index(tuple(dims)[2:], int(flat)), int(flat))


class DenseTensor:
    """Host float64 column-major d-way array (reference DenseTensor)."""

    __slots__ = ("array",)

    def __init__(self, array, dims=None, copy=True):
        a = np.asarray(array, dtype=np.float64)
        if dims is not None:
            a = a.reshape(tuple(int(n) for n in dims), order="F")
        if a.ndim == 0:
            raise ValueError("a tensor needs at least one mode")
        if min(a.shape) < 1:
            raise ValueError(f"every extent must be positive, got {a.shape}")
        a = a.copy(order="F") if copy else np.asfortranarray(a)
        object.__setattr__(self, "array", a)

    def __setattr__(self, name, value):
        raise AttributeError("DenseTensor is read-only")

    @classmethod
    def zeros(cls, dims):
        return cls(np.zeros(tuple(int(n) for n in dims), order="F"), copy=False)

    dims = property(lambda self: self.array.shape)
    ndim = property(lambda self: self.array.ndim)
    size = property(lambda self: self.array.size)

    @property
    def data(self) -> np.ndarray:
        return self.array.reshape(-1, order="F")

    @property
    def slice_shape(self):
        if self.ndim < 2:
            raise ValueError("frontal slices need at least two modes")
        return self.dims[0], self.dims[1]

    @property
    def num_slices(self) -> int:
        if self.ndim < 2:
            raise ValueError("frontal slices need at least two modes")
        return prod(self.dims[2:])

    def slices(self) -> np.ndarray:
        m, p = self.slice_shape
        return self.array.reshape((m, p, self.num_slices), order="F")

    def frontal_slice(self, index) -> np.ndarray:
        flat = index.flat if isinstance(index, SliceIndex) else int(index)
        n = self.num_slices
        if flat < 0 or flat >= n:
            raise IndexError(f"slice {flat} out of range [0, {n})")
        return self.slices()[:, :, flat]

    def unfold(self, mode) -> np.ndarray:
        mode = int(mode)
        if mode < 0 or mode >= self.ndim:
            raise ValueError(f"mode {mode} out of range for {self.ndim} modes")
        return np.reshape(np.moveaxis(self.array, mode, 0), (self.dims[mode], -1), order="F")

    def frobenius_norm(self) -> float:
        return float(np.linalg.norm(self.data))

    def copy(self) -> "DenseTensor":
        return DenseTensor(self.array, copy=True)

    def to_device(self, device=None) -> "DeviceTensor":
        return DeviceTensor.from_host(self, device)

    def __repr__(self):
        return f"DenseTensor(dims={self.dims})"


def refold(matrix, mode, dims) -> DenseTensor:
    """Inverse of DenseTensor.unfold (tensor.py:176-188)."""
    dims = tuple(int(n) for n in dims)
    mode = int(mode)
    if mode < 0 or mode >= len(dims):
        raise ValueError(f"mode {mode} out of range for {len(dims)} modes")
    mat = np.asarray(matrix, dtype=np.float64)
    want = (dims[mode], prod(dims) // dims[mode])
    if mat.shape != want:
        raise ValueError(f"unfolding shape {mat.shape} does not match {want}")
    rest = dims[:mode] + dims[mode + 1:]
    return DenseTensor(np.moveaxis(np.reshape(mat, (dims[mode],) + rest, order="F"), 0, mode))


class DeviceTensor:
    """HBM-resident float64 column-major tensor: ``data`` is a contiguous 1-D
    torch CUDA tensor of prod(dims) elements."""

    __slots__ = ("data", "dims")

    def __init__(self, data, dims):
        import torch
        dims = tuple(int(n) for n in dims)
        if not isinstance(data, torch.Tensor) or data.device.type != "cuda":
            raise TypeError("DeviceTensor data must be a torch CUDA tensor")
        if data.dtype != torch.float64:
            raise TypeError(f"DeviceTensor data must be float64, got {data.dtype}")
        if len(dims) == 0 or min(dims) < 1:
            raise ValueError(f"every extent must be positive, got {dims}")
        if data.numel() != prod(dims):
            raise ValueError(f"{data.numel()} elements for dims {dims}")
        self.data = data.reshape(-1)
        if not self.data.is_contiguous():
            self.data = self.data.contiguous()
        self.dims = dims

    @classmethod
    def from_host(cls, t, device=None, non_blocking=False):
        """Upload a DenseTensor or an array.  A float32 array crosses PCIe as
        float32 and is upcast on the device (starm_upcast_f32_f64): the
        reference's DenseTensor upcast (tensor.py:87) at half the H2D bytes."""
        import torch
        if not isinstance(t, DenseTensor):
            raw = np.asarray(t)
            if raw.dtype == np.float32:
                from . import _native as nat
                dev = torch.device(device or "cuda")
                h32 = torch.from_numpy(np.ascontiguousarray(raw.reshape(-1, order="F")))
                d32 = h32.to(dev, non_blocking=non_blocking)
                out = torch.empty(d32.numel(), dtype=torch.float64, device=dev)
                nat.call("starm_upcast_f32_f64", d32.data_ptr(), out.data_ptr(), d32.numel(),
                         nat.stream_ptr(dev))
                return cls(out, raw.shape)
        arr = t.data if isinstance(t, DenseTensor) else np.asarray(t, dtype=np.float64).reshape(-1, order="F")
        dims = t.dims if isinstance(t, DenseTensor) else np.asarray(t).shape
        host = torch.from_numpy(np.ascontiguousarray(arr))
        return cls(host.to(device or "cuda", non_blocking=non_blocking), dims)

    @classmethod
    def empty(cls, dims, device=None):
        import torch
        return cls(torch.empty(prod(dims), dtype=torch.float64, device=device or "cuda"), dims)

    ndim = property(lambda self: len(self.dims))
    size = property(lambda self: prod(self.dims))
    device = property(lambda self: self.data.device)

    @property
    def slice_shape(self):
        if len(self.dims) < 2:
            raise ValueError("frontal slices need at least two modes")
        return self.dims[0], self.dims[1]

    @property
    def num_slices(self) -> int:
        return prod(self.dims[2:])

    def frobenius_norm(self) -> float:
        return float(self.data.norm())

    def to_host(self) -> DenseTensor:
        arr = device_to_host(self.data)
        return DenseTensor(arr, self.dims, copy=False)

    def __repr__(self):
        return f"DeviceTensor(dims={self.dims}, device={self.data.device})"


PINNED_RESULT_MIN_BYTES = 32 << 20   # larger device-to-host results land in page-locked memory


def device_to_host(*tensors):
    """Device tensors -> numpy arrays (one array for one tensor, else a tuple).
    Large results are copied into page-locked host memory from torch's caching
    host allocator (the arrays are views of it and keep it alive): the copy
    runs at PCIe rate instead of the pageable path's staging plus first-touch
    page faults (c4's 7.3 GB of factors: ~3.5 s pageable).  Falls back to the
    pageable copy if the page-locked allocation fails."""
    import torch
    outs, pending = [], False
    for t in tensors:
        if t.numel() * t.element_size() >= PINNED_RESULT_MIN_BYTES and \
                os.environ.get("STARM_PINNED_RESULTS", "1") != "0":
            try:
                h = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
                h.copy_(t, non_blocking=True)
                outs.append(h)
                pending = True
                continue
            except RuntimeError:
                pass
        outs.append(t.cpu())
    if pending:
        torch.cuda.current_stream(tensors[0].device).synchronize()
    arrs = tuple(o.numpy() for o in outs)
    return arrs[0] if len(arrs) == 1 else arrs


def is_device(t) -> bool:
    return isinstance(t, DeviceTensor)


def as_device(t, device=None) -> DeviceTensor:
    if isinstance(t, DeviceTensor):
        return t
    if isinstance(t, DenseTensor):
        return DeviceTensor.from_host(t, device)
    raise TypeError(f"expected DenseTensor or DeviceTensor, got {type(t).__name__}")
