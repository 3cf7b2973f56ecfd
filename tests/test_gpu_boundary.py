"""GPU parity of the C-ABI entry points added for SURVEY 8(b): the fused
reconstruction + error (starm_reconstruct_f64, K9 + inverse transform +
K10; reference tsvdm.py:342-357 and tests/helpers.py:44-47), the float32
twins (starm_ttm_f32, starm_upcast_f32_f64; reference ttm.py:113-135 and the
tensor.py:87 upcast)."""

import math

import numpy as np
import pytest

import oracle
import paper_2605_16058_b200 as sb
from paper_2605_16058_b200 import _native as nat
from helpers import random_array, random_orthonormal, rel_error

pytestmark = pytest.mark.gpu


def _ref_reconstruct(c, mats):
    f = c.factors.to_host() if hasattr(c.factors, "to_host") else c.factors
    return oracle.reconstruct_packed(c.dims, mats, f.ranks, f.u_data, f.g_data)


@pytest.mark.parametrize("kind,dims,eps", [("dct", (30, 44, 64), 0.3), ("dct", (20, 33, 512), 0.2),
                                           ("custom", (25, 18, 40), 0.1),
                                           ("custom", (16, 40, 24), 0.02)])
def test_fused_reconstruct_matches_reference(kind, dims, eps):
    a = random_array(dims, 3 + dims[2])
    a += 4.0 * np.einsum("i,j,k->ijk", *(np.random.default_rng(1).standard_normal(d) for d in dims))
    t = sb.DenseTensor(a)
    if kind == "dct":
        ts = sb.TransformSet.build(dims, "dct")
    else:
        ts = sb.TransformSet((sb.validate_transform(random_orthonormal(dims[2], 9)),))
    mats = [tr.matrix for tr in ts]
    x = sb.DeviceTensor.from_host(t)
    c = sb.tsvdm_tolerance(x, ts, eps)
    rec, err = sb.reconstruct_fused(c, a=x)
    ref = _ref_reconstruct(c, mats)
    assert rel_error(ref, rec.to_host().array) <= 1e-12
    ref_err = rel_error(a, ref)
    assert abs(err - ref_err) <= 1e-10 * max(ref_err, 1e-300)
    assert abs(err - c.relative_error()) <= 1e-8
    # the public reconstruct routes through it for small nnz and agrees
    rec2 = sb.reconstruct(c.to_host())
    assert rel_error(ref, rec2.array) <= 1e-12


def test_fused_reconstruct_all_ranks_zero_and_explicit_inverse():
    dims = (12, 9, 16)
    a = random_array(dims, 4)
    t = sb.DenseTensor(a)
    ts = sb.TransformSet((sb.validate_transform(random_orthonormal(16, 2)),))
    x = sb.DeviceTensor.from_host(t)
    c = sb.tsvdm_tolerance(x, ts, 0.999)
    if c.factors.total_rank == 0:
        rec, err = sb.reconstruct_fused(c, a=x)
        assert not rec.to_host().array.any() and abs(err - 1.0) <= 1e-15
    # explicit non-orthonormal inverse (the config-4 restatement): out = M^-1 x3 Chat
    rng = np.random.default_rng(5)
    mm = np.eye(16) + 0.1 * rng.standard_normal((16, 16)) / 4
    minv = np.linalg.inv(mm)
    c2 = sb.tsvdm_fixed_rank(x, ts, 3)
    rec, _ = sb.reconstruct_fused(c2, minv=minv)
    f = c2.factors.to_host()
    chat = oracle.reconstruct_packed(dims, [np.eye(16)], f.ranks, f.u_data, f.g_data)
    assert rel_error(oracle.ttm(chat, 2, minv), rec.to_host().array) <= 1e-12


def test_fused_reconstruct_c2_shaped():
    """c2-like fibres (DCT over 1024 time steps): the K = nnz dense product
    with the reference's own M^T columns."""
    from paper_2605_16058_b200 import configs as cf
    a = cf.config2(nlat=46, nlon=90, nt=1024, seed=1)
    t = sb.DenseTensor(a)
    ts = sb.TransformSet.build(a.shape, "dct")
    x = sb.DeviceTensor.from_host(t)
    c = sb.tsvdm_tolerance(x, ts, 1e-2)
    nnz = int((c.factors.to_host().ranks > 0).sum())
    assert 0 < nnz
    rec, err = sb.reconstruct_fused(c, a=x)
    ref = _ref_reconstruct(c, [tr.matrix for tr in ts])
    assert rel_error(ref, rec.to_host().array) <= 1e-12
    assert abs(err - rel_error(a, ref)) <= 1e-10 * err
    assert abs(err - c.relative_error()) <= 1e-8 and err <= 1e-2


@pytest.mark.parametrize("rows,inner,batch,out_cols", [(7, 5, 1, 3), (64, 33, 3, 40),
                                                        (1000, 128, 2, 128)])
def test_ttm_f32_twin(rows, inner, batch, out_cols):
    import torch
    rng = np.random.default_rng(rows)
    src = rng.standard_normal(rows * inner * batch).astype(np.float32)
    mat = rng.standard_normal((out_cols, inner)).astype(np.float32)
    lib = nat.load()
    nbytes = lib.starm_ttm_f32_workspace_bytes(rows, inner, batch, out_cols)
    ws = nat.workspace(nbytes, "cuda")
    xs = torch.from_numpy(src).cuda()
    xm = torch.from_numpy(np.ascontiguousarray(mat)).cuda()
    out = torch.empty(rows * out_cols * batch, dtype=torch.float32, device="cuda")
    nat.call("starm_ttm_f32", xs.data_ptr(), xm.data_ptr(), out.data_ptr(), rows, inner, batch,
             out_cols, ws.data_ptr(), nbytes, nat.stream_ptr())
    got = out.cpu().numpy()
    # reference: f32 operands upcast (tensor.py:87), f64 product, one rounding to f32
    ref = np.concatenate([
        (mat.astype(np.float64) @ src[b * rows * inner:(b + 1) * rows * inner].astype(np.float64)
         .reshape(inner, rows)).ravel() for b in range(batch)])
    assert np.max(np.abs(got - ref.astype(np.float32))) <= 1e-6 * np.max(np.abs(ref))
    assert rel_error(ref, got.astype(np.float64)) <= 1e-7


def test_float32_input_upcast_on_device():
    a32 = np.asfortranarray(np.random.default_rng(2).standard_normal((17, 9, 5)).astype(np.float32))
    x = sb.DeviceTensor.from_host(a32)
    assert x.dims == a32.shape
    assert np.array_equal(x.to_host().array, a32.astype(np.float64))
    # same result as the host upcast of the reference's DenseTensor
    ts = sb.TransformSet.build(a32.shape, "dct")
    c1 = sb.tsvdm_tolerance(x, ts, 0.3)
    c2 = sb.tsvdm_tolerance(sb.DenseTensor(a32), ts, 0.3)
    assert np.array_equal(c1.to_host().ranks, c2.ranks)
    assert c1.discarded_energy == c2.discarded_energy


# ------------------------------------------------------------------ block-wise host upload
# tsvdm_tolerance(DenseTensor) cuts the fibres into runs and transforms run g
# behind the host-to-device copy of run g+1 (starm_copy2d_h2d,
# starm_dct_pack_block_f64, starm_slice_energy_block_f64).  Every fibre goes
# through the same kernel as in the one-shot path, so the transform-domain
# tensor and the bf16 operand must be BITWISE those of starm_dct_pack_f64 and
# the compression result identical to the device-resident call
# (reference: to_transform_domain, ttm.py:138-144, then tsvdm.py:268-321).

@pytest.mark.parametrize("dims,blocks", [((40, 52, 1024), 5), ((37, 21, 1024), 3), ((16, 24, 256), 2),
                                         ((9, 31, 512), 16)])
def test_blockwise_upload_is_bitwise_the_one_shot_transform(dims, blocks):
    import torch
    from paper_2605_16058_b200.mode_product import DeferredResidual
    a = random_array(dims, 11 + dims[0])
    t = sb.DenseTensor(a)
    ts = sb.TransformSet.build(dims, "dct")
    dev = nat.require_cuda()
    one = DeferredResidual(sb.DeviceTensor.from_host(t), ts[0])
    blk = DeferredResidual.from_host(t, ts[0], dev, blocks=blocks)
    torch.cuda.synchronize()
    assert torch.equal(one.out.data, blk.out.data)
    nb = nat.load().starm_ttm_residual_workspace_bytes(dims[0] * dims[1], dims[2], 1)
    off1 = one.base - one._ws.data_ptr()
    off2 = blk.base - blk._ws.data_ptr()
    rows = dims[0] * dims[1]
    live = rows * dims[2] * 2          # the live operand rows (pad rows are never read past TMA bounds)
    assert torch.equal(one._ws[off1:off1 + live], blk._ws[off2:off2 + live])
    assert nb >= live
    # partial energies summed over the runs = the per-slice energies
    f = torch.empty(dims[2], dtype=torch.float64, device=dev)
    nat.call("starm_slice_energy_f64", one.out.data.data_ptr(), rows, dims[2], f.data_ptr(),
             nat.stream_ptr(dev))
    ref = (np.asarray(one.out.data.cpu()).reshape(dims[2], rows) ** 2).sum(axis=1)
    assert np.allclose(blk.energies.cpu().numpy(), ref, rtol=1e-13)
    assert np.allclose(f.cpu().numpy(), ref, rtol=1e-13)


def test_blockwise_upload_compression_equals_device_resident_call(monkeypatch):
    import os
    import torch
    from paper_2605_16058_b200 import mode_product as mp_
    if os.environ.get("STARM_PIPELINE", "1") == "0":
        pytest.skip("STARM_PIPELINE=0")
    dims = (48, 40, 1024)
    rng = np.random.default_rng(5)
    tt = np.arange(dims[2])
    a = sum(np.einsum("i,j,k->ijk", rng.standard_normal(dims[0]), rng.standard_normal(dims[1]),
                      np.cos(2 * np.pi * (q + 1) * tt / dims[2] + rng.uniform(0, 6.28)))
            for q in range(5))
    a = np.asfortranarray(a + 1e-2 * rng.standard_normal(dims))
    t = sb.DenseTensor(a)
    ts = sb.TransformSet.build(dims, "dct")
    ref = sb.tsvdm_tolerance(sb.DeviceTensor.from_host(t), ts, 2e-2)
    monkeypatch.setattr(mp_, "PIPELINE_MIN_BYTES", 0)
    monkeypatch.setattr(mp_, "PIPELINE_BLOCKS", 4)
    assert mp_.pipelined_upload_applies(t, ts)
    got = sb.tsvdm_tolerance(t, ts, 2e-2)          # host in -> host out, block-wise upload
    rf = ref.factors.to_host()
    assert np.array_equal(got.ranks, ref.ranks)
    assert np.array_equal(got.factors.u_data, rf.u_data)
    assert np.array_equal(got.factors.g_data, rf.g_data)
    assert abs(got.total_energy - ref.total_energy) <= 1e-13 * ref.total_energy
    assert abs(got.discarded_energy - ref.discarded_energy) <= 1e-12 * ref.total_energy
    mats = [tr.matrix for tr in ts]
    o = oracle.tsvdm_tolerance(a, mats, 2e-2)
    assert np.array_equal(got.ranks, o["ranks"])


def test_blockwise_dense_upload_equals_device_resident_fixed_rank(monkeypatch):
    """Dense (Haar) transform: the host call uploads fibre runs and multiplies
    each behind the next copy (starm_ttm_block_f64); bitwise the one-shot
    forward product, so the fixed-rank result equals the device-resident one
    (reference: ttm.py:113-135 then tsvdm.py:246-265)."""
    import os
    import torch
    from paper_2605_16058_b200 import mode_product as mp_
    if os.environ.get("STARM_PIPELINE", "1") == "0":
        pytest.skip("STARM_PIPELINE=0")
    dims = (45, 37, 96)
    a = random_array(dims, 17)
    t = sb.DenseTensor(a)
    ts = sb.TransformSet((sb.validate_transform(random_orthonormal(dims[2], 3)),))
    dev = nat.require_cuda()
    one = mp_.forward_device(sb.DeviceTensor.from_host(t), ts)
    monkeypatch.setattr(mp_, "PIPELINE_MIN_BYTES", 0)
    monkeypatch.setattr(mp_, "PIPELINE_BLOCKS", 5)
    blk = mp_.forward_from_host(t, ts, dev)
    assert blk is not None
    torch.cuda.synchronize()
    assert torch.equal(one.data, blk.data)
    ref = sb.tsvdm_fixed_rank(sb.DeviceTensor.from_host(t), ts, 6)
    got = sb.tsvdm_fixed_rank(t, ts, 6)
    rf = ref.factors.to_host()
    assert np.array_equal(got.factors.u_data, rf.u_data) and np.array_equal(got.factors.g_data, rf.g_data)
    assert got.discarded_energy == ref.discarded_energy and got.total_energy == ref.total_energy
    o = oracle.tsvdm_fixed_rank(a, [ts[0].matrix], 6)
    assert abs(got.discarded_energy - o["discarded_energy"]) <= 1e-12 * o["total_energy"]
    # the DCT kind below the FFT threshold (n = 64: dense product with tr.matrix) qualifies too
    ts2 = sb.TransformSet.build((45, 37, 64), "dct")
    t2 = sb.DenseTensor(random_array((45, 37, 64), 18))
    one2 = mp_.forward_device(sb.DeviceTensor.from_host(t2), ts2)
    blk2 = mp_.forward_from_host(t2, ts2, dev)
    assert blk2 is not None and torch.equal(one2.data, blk2.data)


def test_large_results_return_in_page_locked_buffers(monkeypatch):
    """device_to_host: results above the size floor are copied into page-locked
    buffers (numpy views that keep them alive), smaller ones take the
    pageable copy; values are the same either way."""
    import os
    import torch
    from paper_2605_16058_b200 import tensors as tn
    if os.environ.get("STARM_PINNED_RESULTS", "1") == "0":
        pytest.skip("STARM_PINNED_RESULTS=0")
    dev = nat.require_cuda()
    x = torch.arange(1 << 16, dtype=torch.float64, device=dev)
    y = torch.arange(7, dtype=torch.float64, device=dev)
    monkeypatch.setattr(tn, "PINNED_RESULT_MIN_BYTES", 1 << 18)
    a, b = tn.device_to_host(x, y)
    assert np.array_equal(a, np.arange(1 << 16, dtype=np.float64)) and np.array_equal(b, np.arange(7.0))
    assert torch.from_numpy(a).is_pinned() and not torch.from_numpy(b).is_pinned()
    monkeypatch.setenv("STARM_PINNED_RESULTS", "0")
    c = tn.device_to_host(x)
    assert np.array_equal(c, a) and not torch.from_numpy(c).is_pinned()
    # a compression whose factors exceed the floor comes back identical
    monkeypatch.delenv("STARM_PINNED_RESULTS")
    monkeypatch.setattr(tn, "PINNED_RESULT_MIN_BYTES", 1 << 10)
    dims = (40, 36, 32)
    t = sb.DenseTensor(random_array(dims, 5))
    ts = sb.TransformSet.build(dims, "dct")
    got = sb.tsvdm_fixed_rank(t, ts, 7)
    monkeypatch.setattr(tn, "PINNED_RESULT_MIN_BYTES", 1 << 40)
    ref = sb.tsvdm_fixed_rank(t, ts, 7)
    assert np.array_equal(got.factors.u_data, ref.factors.u_data)
    assert np.array_equal(got.factors.g_data, ref.factors.g_data)
