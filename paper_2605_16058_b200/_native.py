"""ctypes binding of ``libstarm.so`` (the sm_100a C ABI declared in
``include/starm.h``).

The library is the only compute path: there is no CPU fallback.  If the
shared object is missing, or no CUDA device is present, every compute entry
point raises immediately.  ``ctypes.CDLL`` releases the GIL for the
duration of each foreign call.
"""

from __future__ import annotations

import ctypes
import os
from ctypes import c_double, c_int, c_int64, c_size_t, c_void_p

import numpy as np

_LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libstarm.so")

OK = 0
INVALID_ARG = 1
NONFINITE_SLICE = 2
NOCONVERGE = 3
CUDA_ERROR = 4
UNSUPPORTED = 5

SVD_VALUES = 0
SVD_FULL = 1
SVD_TRUNCATED = 2
SVD_VALUES_STATE = 3
SVD_TRUNCATED_STATE = 4

# name -> (restype, argtypes); mirrors include/starm.h one-to-one.
SIGNATURES = {
    "starm_abi_version": (c_int, []),
    "starm_last_error": (c_size_t, [ctypes.c_char_p, c_size_t]),
    "starm_ttm_f64": (c_int, [c_void_p, c_void_p, c_void_p, c_int64, c_int64, c_int64, c_int64,
                              c_void_p]),
    "starm_ttm_block_f64": (c_int, [c_void_p, c_void_p, c_void_p, c_int64, c_int64, c_int64, c_int64,
                                    c_int64, c_void_p]),
    "starm_dct_f64": (c_int, [c_void_p, c_void_p, c_int64, c_int64, c_int64, c_int, c_void_p]),
    "starm_facewise_gemm_f64": (c_int, [c_void_p, c_void_p, c_void_p, c_int64, c_int64, c_int64,
                                        c_int64, c_void_p]),
    "starm_svd_workspace_bytes": (c_size_t, [c_int64, c_int64, c_int64, c_int64, c_int]),
    "starm_svd_f64": (c_int, [c_void_p, c_int64, c_int64, c_int64, c_void_p, c_int64, c_int,
                              c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
                              c_void_p, c_void_p, c_void_p, c_void_p, c_size_t, c_void_p]),
    "starm_threshold_workspace_bytes": (c_size_t, [c_int64, c_int64]),
    "starm_threshold_f64": (c_int, [c_void_p, c_int64, c_int64, c_double, c_void_p, c_void_p,
                                    c_void_p, c_void_p, c_void_p, c_void_p, c_size_t, c_void_p]),
    "starm_pack_offsets": (c_int, [c_void_p, c_int64, c_int64, c_int64, c_void_p, c_void_p,
                                   c_void_p]),
    "starm_unpack_facewise_f64": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
                                          c_int64, c_int64, c_int64, c_void_p, c_void_p]),
    "starm_error_sums_workspace_bytes": (c_size_t, [c_int64]),
    "starm_error_sums_f64": (c_int, [c_void_p, c_void_p, c_int64, c_void_p, c_void_p, c_size_t,
                                     c_void_p]),
    "starm_pack_from_full_f64": (c_int, [c_void_p, c_void_p, c_void_p, c_int64, c_int64, c_int64,
                                         c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
                                         c_void_p]),
    "starm_tail_energy_f64": (c_int, [c_void_p, c_int64, c_int64, c_int64, c_void_p, c_void_p]),
    "starm_ttm_residual_workspace_bytes": (c_size_t, [c_int64, c_int64, c_int64]),
    "starm_ttm_residual_bf16": (c_int, [c_void_p, c_void_p, c_int, c_void_p, c_int64, c_int64,
                                        c_int64, c_void_p, c_size_t, c_void_p]),
    "starm_reconstruct_workspace_bytes": (c_size_t, [c_int64, c_int64, c_int64, c_int64]),
    "starm_reconstruct_f64": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_int64,
                                      c_int64, c_int64, c_void_p, c_int64, c_void_p, c_void_p,
                                      c_void_p, c_void_p, c_void_p, c_size_t, c_void_p]),
    "starm_ttm_f32_workspace_bytes": (c_size_t, [c_int64, c_int64, c_int64, c_int64]),
    "starm_ttm_f32": (c_int, [c_void_p, c_void_p, c_void_p, c_int64, c_int64, c_int64, c_int64,
                              c_void_p, c_size_t, c_void_p]),
    "starm_upcast_f32_f64": (c_int, [c_void_p, c_void_p, c_int64, c_void_p]),
    "starm_dct_residual_f64": (c_int, [c_void_p, c_void_p, c_int64, c_int64, c_int64, c_int,
                                       c_void_p, c_int, c_void_p, c_size_t, c_void_p]),
    "starm_threshold_pruned_f64": (c_int, [c_void_p, c_int64, c_int64, c_double, c_double,
                                           c_double, c_void_p, c_void_p, c_void_p, c_void_p,
                                           c_void_p, c_size_t, c_void_p]),
    "starm_slice_energy_f64": (c_int, [c_void_p, c_int64, c_int64, c_void_p, c_void_p]),
    "starm_dct_pack_f64": (c_int, [c_void_p, c_void_p, c_int64, c_int64, c_int64, c_int,
                                   c_void_p, c_size_t, c_void_p]),
    "starm_dct_pack_block_f64": (c_int, [c_void_p, c_void_p, c_int64, c_int64, c_int64, c_int64,
                                         c_void_p, c_size_t, c_void_p]),
    "starm_slice_energy_block_f64": (c_int, [c_void_p, c_int64, c_int64, c_int64, c_int64,
                                             c_void_p, c_void_p]),
    "starm_copy2d_h2d": (c_int, [c_void_p, c_size_t, c_void_p, c_size_t, c_size_t, c_size_t,
                                 c_void_p]),
    "starm_residual_apply_f64": (c_int, [c_void_p, c_void_p, c_int, c_void_p, c_int64, c_int64,
                                         c_int64, c_int64, c_void_p]),
    "starm_gram_workspace_bytes": (c_size_t, [c_int64, c_int64, c_int64]),
    "starm_gram_f64": (c_int, [c_void_p, c_int64, c_int64, c_int64, c_void_p, c_void_p, c_size_t,
                               c_void_p]),
    "starm_launch_count_reset": (ctypes.c_longlong, []),
    "starm_svd_tune": (c_int, [c_int, c_int, c_int, c_int]),
    "starm_svd_stats": (c_int, [c_void_p, c_int]),
}

SVD_STAT_NAMES = ("slices", "sweeps", "pairs", "rotated", "cyc_gram", "cyc_eig", "cyc_apply",
                  "cyc_qr", "cyc_final", "cyc_load", "cyc_band", "cyc_bulge", "cyc_pfact",
                  "cyc_trail", "cyc_right", "cyc_pmisc")


def svd_stats(reset=True) -> dict:
    """Diagnostic counters of the Jacobi kernels (enable with
    ``load().starm_svd_tune(-1, -1, -1, 1)``)."""
    buf = (ctypes.c_ulonglong * 16)()
    check(load().starm_svd_stats(ctypes.addressof(buf), int(reset)), "starm_svd_stats")
    return {k: int(buf[i]) for i, k in enumerate(SVD_STAT_NAMES)}

_lib = None


class NativeLibraryMissing(RuntimeError):
    pass


def library_path() -> str:
    return _LIB_PATH


def load():
    """Load libstarm.so (idempotent).  Raises if it has not been built."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(_LIB_PATH):
        raise NativeLibraryMissing(
            f"{_LIB_PATH} not found: build it with `make` (or __graft_entry__.build()); "
            "the t-SVDM path has no CPU fallback"
        )
    lib = ctypes.CDLL(_LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def last_error() -> str:
    lib = load()
    buf = ctypes.create_string_buffer(2048)
    lib.starm_last_error(buf, 2048)
    return buf.value.decode(errors="replace")


def check(status: int, what: str):
    if status == OK:
        return
    msg = f"{what}: {last_error()}"
    if status in (INVALID_ARG, UNSUPPORTED, NONFINITE_SLICE):
        raise ValueError(msg)
    if status == NOCONVERGE:
        raise np.linalg.LinAlgError(msg)
    raise RuntimeError(msg)


_STREAM_DEVICE = {}  # cudaStream_t handle -> device index (filled by stream_ptr)


def call(name: str, *args):
    """Invoke a C-ABI entry point.  Calls whose last argument is a stream
    handle from ``stream_ptr`` run with that stream's device current, so
    tensors on cuda:N work while another device is current (the library's
    per-device tables, attributes and side streams key off cudaGetDevice)."""
    lib = load()
    dev = _STREAM_DEVICE.get(args[-1]) if args and isinstance(args[-1], int) else None
    if dev is not None:
        t = torch()
        if t.cuda.current_device() != dev:
            with t.cuda.device(dev):
                check(getattr(lib, name)(*args), name)
            return
    check(getattr(lib, name)(*args), name)


# ------------------------------------------------------------------ device

def torch():
    import torch as _torch
    return _torch


def require_cuda(device=None):
    """Return the torch.device the computation runs on; raise without CUDA."""
    t = torch()
    if not t.cuda.is_available():
        raise RuntimeError(
            "paper_2605_16058_b200 needs a CUDA (sm_100a) device; there is no CPU fallback"
        )
    load()
    if device is None:
        return t.device("cuda", t.cuda.current_device())
    dev = t.device(device)
    if dev.type != "cuda":
        raise ValueError(f"device must be a CUDA device, got {dev}")
    if dev.index is None:
        dev = t.device("cuda", t.cuda.current_device())
    return dev


def stream_ptr(device=None) -> int:
    t = torch()
    st = t.cuda.current_stream(device)
    h = st.cuda_stream
    if h not in _STREAM_DEVICE or _STREAM_DEVICE[h] != st.device.index:
        _STREAM_DEVICE[h] = st.device.index
    return h


def register_stream(stream) -> int:
    """Handle of an explicit torch stream, registered so ``call`` runs its
    launches with the stream's device current."""
    h = stream.cuda_stream
    _STREAM_DEVICE[h] = stream.device.index
    return h


def ptr(x) -> int:
    return 0 if x is None else x.data_ptr()


def empty(n, dtype=None, device=None):
    t = torch()
    return t.empty(int(n), dtype=dtype or t.float64, device=device)


def workspace(nbytes: int, device=None):
    t = torch()
    return t.empty(max(int(nbytes), 16), dtype=t.uint8, device=device)
