"""Host-side logic of the drop-in API and the C ABI surface (no GPU needed).

Mirrors the reference's host-only tests (tests/test_tensor.py,
test_transforms.py, the validation halves of test_ttm.py / test_tsvdm.py /
test_slicesvd.py): everything here runs before any device work."""

import ctypes
import math
import os
import re

import numpy as np
import pytest

import paper_2605_16058_b200 as sb
from paper_2605_16058_b200 import _native
from tests.golden.cases import random_orthonormal

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


# ------------------------------------------------------------------ C ABI

def _header_symbols():
    text = open(os.path.join(ROOT, "include", "starm.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(starm_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_header_symbol():
    lib = ctypes.CDLL(_native.library_path())
    syms = _header_symbols()
    assert len(syms) >= 15
    for name in syms:
        assert hasattr(lib, name), name
    assert set(syms) == set(_native.SIGNATURES), set(syms) ^ set(_native.SIGNATURES)


def test_abi_version_and_error_channel():
    lib = _native.load()
    assert lib.starm_abi_version() == 1
    # invalid arguments are rejected before any device work
    rc = lib.starm_ttm_f64(None, None, None, 0, 4, 1, 4, None)
    assert rc == _native.INVALID_ARG
    assert "extents" in _native.last_error()
    with pytest.raises(ValueError):
        _native.check(rc, "starm_ttm_f64")
    rc = lib.starm_threshold_f64(None, 3, 4, 1.5, None, None, None, None, None, None, 0, None)
    assert rc == _native.INVALID_ARG and "tolerance" in _native.last_error()


def test_status_mapping():
    with pytest.raises(np.linalg.LinAlgError):
        _native.check(_native.NOCONVERGE, "x")
    with pytest.raises(RuntimeError):
        _native.check(_native.CUDA_ERROR, "x")


# ----------------------------------------------------------------- tensor

def test_linear_index_and_bijection():
    assert sb.linear_index((3, 4, 2), (1, 2, 1)) == 19
    dims = (3, 4, 2, 2)
    seen = set()
    for idx in np.ndindex(*dims):
        off = sb.linear_index(dims, idx)
        assert sb.multi_index(dims, off) == idx
        seen.add(off)
    assert seen == set(range(48))
    with pytest.raises(IndexError):
        sb.linear_index((3, 4), (3, 0))
    with pytest.raises(ValueError):
        sb.linear_index((3, 4), (1,))


def test_dense_tensor_layout():
    t = sb.DenseTensor(np.arange(8.0), (2, 2, 2), copy=False)
    assert np.array_equal(t.frontal_slice(1), [[4, 6], [5, 7]])
    assert np.array_equal(t.unfold(2), [[0, 1, 2, 3], [4, 5, 6, 7]])
    si = sb.SliceIndex.from_trailing((2, 2, 3, 2), (2, 1))
    assert si.flat == 5
    t4 = sb.DenseTensor(np.arange(24.0), (2, 2, 3, 2))
    assert np.array_equal(t4.frontal_slice(si).reshape(-1, order="F"), np.arange(20.0, 24.0))
    f32 = sb.DenseTensor(np.ones((2, 2, 2), dtype=np.float32))
    assert f32.array.dtype == np.float64 and f32.array.flags.f_contiguous
    with pytest.raises(AttributeError):
        t.array = None
    with pytest.raises(IndexError):
        t.frontal_slice(2)
    back = sb.refold(t4.unfold(3), 3, t4.dims)
    assert np.array_equal(back.array, t4.array)


# ------------------------------------------------------------- transforms

def test_dct_and_validation():
    m = sb.dct_matrix(2).matrix
    assert np.allclose(m, [[math.sqrt(0.5)] * 2, [math.cos(math.pi / 4), math.cos(3 * math.pi / 4)]],
                       atol=1e-15)
    for n in (1, 3, 16, 257):
        assert sb.orthonormality_residual(sb.dct_matrix(n).matrix) <= 1e-10
    with pytest.raises(ValueError, match="residual"):
        sb.validate_transform(2.0 * np.eye(4))
    with pytest.raises(ValueError):
        sb.validate_transform(np.zeros((3, 4)))
    with pytest.raises(ValueError):
        sb.Transform(np.eye(3), "fourier")
    with pytest.raises(TypeError):
        sb.TransformSet((np.eye(3),))
    ts = sb.TransformSet.build((3, 4, 5, 6), ["dct", sb.validate_transform(random_orthonormal(6, 1))])
    assert ts.kinds == ("dct", "custom") and ts.sizes == (5, 6)
    with pytest.raises(ValueError):
        ts.check_dims((3, 4, 5, 7))
    with pytest.raises(ValueError):
        sb.TransformSet.build((3, 4, 5), "data-driven")  # needs the tensor


def test_ttm_plan_and_validation():
    plan = sb.TTMPlan.for_dims((3, 4, 5, 6), 2, out_cols=7)
    assert (plan.rows, plan.inner, plan.batch, plan.out_cols) == (12, 5, 6, 7)
    assert not plan.is_last_mode
    assert sb.TTMPlan.for_dims((3, 4, 5, 6), 3, out_cols=6).is_last_mode
    with pytest.raises(ValueError):
        sb.TTMPlan.for_dims((3, 4, 5), 1, out_cols=4)
    with pytest.raises(ValueError):
        sb.TTMPlan.for_dims((3, 4, 5), 2, out_cols=5, variant="vectorized")
    t = sb.DenseTensor(np.ones((3, 4, 5)))
    with pytest.raises(ValueError):
        sb.ttm(t, 1, np.eye(4))
    with pytest.raises(ValueError):
        sb.ttm(t, 2, np.eye(4))
    with pytest.raises(ValueError):
        sb.ttm(t, 2, np.zeros(5))
    with pytest.raises(ValueError):
        sb.ttm(t, 2, np.eye(5), threads=0)


# ------------------------------------------------------- packed factors

def test_variable_rank_factors_container():
    with pytest.raises(ValueError):
        sb.VariableRankFactors(3, 2, np.array([1]), np.zeros(2), np.zeros(2))
    with pytest.raises(ValueError):
        sb.VariableRankFactors(3, 2, np.array([3]), np.zeros(9), np.zeros(6))
    ok = sb.VariableRankFactors(3, 2, np.array([1, 0]), np.zeros(3), np.zeros(2))
    assert ok.u_block(1).shape == (3, 0)
    assert ok.g_block(0).shape == (1, 2)
    f = sb.VariableRankFactors.allocate(4, 5, [2, 0, 1])
    assert f.total_rank == 3 and f.u_data.size == 12 and f.g_data.size == 15


def test_compressed_tensor_validation_and_ratio():
    factors = sb.VariableRankFactors.allocate(10, 10, np.full(10, 10))
    ts = sb.TransformSet((sb.dct_matrix(10),))
    c = sb.CompressedTensor((10, 10, 10), ts, factors, "tsvdm1", 10.0)
    assert sb.compression_ratio(c) == 0.5
    with pytest.raises(ValueError):
        sb.CompressedTensor((10, 10, 11), ts, factors, "tsvdm1", 10.0)
    with pytest.raises(ValueError):
        sb.CompressedTensor((10, 10, 10), ts, factors, "tsvdm9", 10.0)
    with pytest.raises(ValueError):
        sb.CompressedTensor((10, 10, 10), ts, sb.VariableRankFactors.allocate(10, 10, np.arange(10)),
                            "tsvdm1", 10.0)
    zero = sb.CompressedTensor((4, 4, 3), sb.TransformSet((sb.identity_transform(3),)),
                               sb.VariableRankFactors.allocate(4, 4, np.zeros(3, dtype=np.int64)),
                               "tsvdm2", 0.5)
    assert sb.compression_ratio(zero) == math.inf
    assert zero.relative_error() is None
    c2 = sb.CompressedTensor((10, 10, 10), ts, factors, "tsvdm1", 10.0, 1.0, 4.0)
    assert c2.relative_error() == 0.5
    dims = (73, 144, 17, 4, 365, 10)
    n = 17 * 4 * 365 * 10
    big = sb.CompressedTensor(dims, sb.TransformSet(tuple(sb.dct_matrix(k) for k in dims[2:])),
                              sb.VariableRankFactors.allocate(73, 144, np.ones(n, dtype=np.int64)),
                              "tsvdm1", 1.0)
    expected = np.prod([float(d) for d in dims]) / (n * (73 + 144))
    assert abs(sb.compression_ratio(big) - expected) <= 1e-9 * expected


def test_argument_validation_precedes_device_work():
    t = sb.DenseTensor(np.ones((4, 5, 3)))
    ts = sb.TransformSet.build(t.dims, "dct")
    with pytest.raises(ValueError):
        sb.tsvdm_fixed_rank(t, ts, 0)
    with pytest.raises(ValueError):
        sb.tsvdm_fixed_rank(t, ts, 5)
    with pytest.raises(ValueError):
        sb.tsvdm_tolerance(t, ts, 1.5)
    with pytest.raises(ValueError):
        sb.tsvdm_tolerance(t, ts, 0.2, strategy="lazy")
    with pytest.raises(ValueError):
        sb.compute_threshold(np.ones((2, 2)), 0.0)
    with pytest.raises(ValueError):
        sb.compute_threshold(-np.ones((2, 2)), 0.5)
    with pytest.raises(ValueError):
        sb.compute_threshold(np.full((2, 2), np.nan), 0.5)
    with pytest.raises(ValueError):
        sb.svd_all_slices(t, strategy="gpu")
    with pytest.raises(ValueError):
        sb.svd_all_slices(t, threads=0)
    with pytest.raises(ValueError):
        sb.svd_truncated_slices(t, np.array([1, 2]))
    with pytest.raises(ValueError):
        sb.starm_product(t, sb.DenseTensor(np.ones((3, 3, 3))), ts)
    with pytest.raises(ValueError):
        sb.tsvdm_tolerance(sb.DenseTensor(np.ones((3, 3))), ts, 0.1)


def test_no_cpu_fallback():
    import torch
    if torch.cuda.is_available():
        pytest.skip("has a GPU")
    t = sb.DenseTensor(np.ones((4, 5, 3)))
    ts = sb.TransformSet.build(t.dims, "dct")
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        sb.tsvdm_tolerance(t, ts, 0.1)
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        sb.ttm(t, 2, np.eye(3))


def test_devices_argument_validation():
    from paper_2605_16058_b200.compress import _resolve_devices
    assert _resolve_devices(None) == (None, None)
    with pytest.raises(ValueError, match="devices"):
        _resolve_devices(3.5)


def test_blockwise_upload_policy(monkeypatch):
    """The block-wise host upload applies to host tensors whose forward
    transform is the deferrable DCT (3-way, power-of-two length >= 256) and
    that are large enough; STARM_PIPELINE=0 switches it off."""
    from paper_2605_16058_b200 import mode_product as mp
    t = sb.DenseTensor(np.zeros((4, 6, 256), order="F"))
    ts = sb.TransformSet.build(t.dims, "dct")
    assert not mp.pipelined_upload_applies(t, ts)            # 48 KB: below the size floor
    monkeypatch.setattr(mp, "PIPELINE_MIN_BYTES", 0)
    assert mp.pipelined_upload_applies(t, ts)
    monkeypatch.setenv("STARM_PIPELINE", "0")
    assert not mp.pipelined_upload_applies(t, ts)
    monkeypatch.delenv("STARM_PIPELINE")
    t64 = sb.DenseTensor(np.zeros((4, 6, 64), order="F"))    # n = 64: dense product, not deferrable
    assert not mp.pipelined_upload_applies(t64, sb.TransformSet.build(t64.dims, "dct"))
    t4 = sb.DenseTensor(np.zeros((4, 6, 2, 256), order="F"))  # 4-way: not the 3-way fast path
    assert not mp.pipelined_upload_applies(t4, sb.TransformSet.build(t4.dims, "dct"))
