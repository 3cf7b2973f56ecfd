"""The sharded pipeline with the CUDA ops (DeviceOps) over NCCL at world size
1 on cuda:0: the collective schedule runs through libstarm kernels and must
reproduce the single-GPU tsvdm_tolerance decision.  (Multi-rank host logic:
tests/test_sharded.py, gloo, world sizes 2 and 3.)"""

import os
import socket

import numpy as np
import pytest

import paper_2605_16058_b200 as sb
from paper_2605_16058_b200.sharded import (DeviceOps, ShardPlan, gather_factors,
                                           reconstruct_sharded, relative_error_sharded,
                                           scatter_fibres, tsvdm_tolerance_sharded)

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.fixture(scope="module")
def nccl_world1():
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(_free_port())
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1)
    yield dist
    dist.destroy_process_group()


@pytest.mark.parametrize("dims,eps", [((37, 41, 64), 0.05), ((60, 20, 16), 0.1)])
def test_sharded_device_ops_match_tsvdm_tolerance(nccl_world1, dims, eps):
    import torch
    dist = nccl_world1
    rng = np.random.default_rng(3)
    a = np.asfortranarray(rng.standard_normal(dims))
    a += np.einsum("i,j,k->ijk", rng.standard_normal(dims[0]), rng.standard_normal(dims[1]),
                   rng.standard_normal(dims[2])) * 5
    dev = torch.device("cuda", 0)
    tr = sb.dct_matrix(dims[2])
    ts = sb.TransformSet((tr,))
    ref = sb.tsvdm_tolerance(sb.DenseTensor(a), ts, eps)
    plan = ShardPlan(dims[0], dims[1], dims[2], 1, 0)
    local = torch.from_numpy(scatter_fibres(a, plan).reshape(-1, order="F").copy()).to(dev)
    ops = DeviceOps(tr, dev)
    res = tsvdm_tolerance_sharded(local, plan, ops, eps, dist)
    assert np.array_equal(res.ranks, ref.ranks)
    assert abs(res.discarded_energy - ref.discarded_energy) <= 1e-12 * ref.total_energy
    assert abs(res.total_energy - ref.total_energy) <= 1e-12 * ref.total_energy
    u, g = gather_factors(res, plan, dist)
    assert u.numel() == ref.factors.u_data.size and g.numel() == ref.factors.g_data.size
    rec = reconstruct_sharded(res, plan, ops, dist)
    err = relative_error_sharded(local, rec, dist)
    assert abs(err - res.relative_error) <= 1e-10
    assert err < eps


def test_dropin_devices_group_matches_single_gpu(nccl_world1):
    """devices="dist" on the drop-in entry points runs the sharded pipeline
    (SPMD over the default process group) and returns the same
    CompressedTensor as the single-device call."""
    dims = (33, 20, 48)
    rng = np.random.default_rng(7)
    a = np.asfortranarray(rng.standard_normal(dims))
    a += np.einsum("i,j,k->ijk", rng.standard_normal(33), rng.standard_normal(20),
                   rng.standard_normal(48)) * 3
    t = sb.DenseTensor(a)
    ts = sb.TransformSet.build(dims, "dct")
    for call in (lambda **kw: sb.tsvdm_tolerance(t, ts, 0.1, **kw),
                 lambda **kw: sb.tsvdm_fixed_rank(t, ts, 4, **kw)):
        ref = call()
        got = call(devices="dist")
        assert np.array_equal(got.ranks, ref.ranks)
        assert abs(got.discarded_energy - ref.discarded_energy) <= 1e-12 * ref.total_energy
        assert abs(got.total_energy - ref.total_energy) <= 1e-12 * ref.total_energy
        assert got.factors.u_data.shape == ref.factors.u_data.shape
        rec = sb.reconstruct(got)
        err = float(np.linalg.norm(rec.data - t.data) / np.linalg.norm(t.data))
        assert abs(err - got.relative_error()) <= 1e-8


def test_dropin_devices_explicit_device():
    dims = (10, 12, 8)
    a = np.asfortranarray(np.random.default_rng(1).standard_normal(dims))
    ts = sb.TransformSet.build(dims, "dct")
    ref = sb.tsvdm_tolerance(sb.DenseTensor(a), ts, 0.2)
    got = sb.tsvdm_tolerance(sb.DenseTensor(a), ts, 0.2, devices=0)
    assert np.array_equal(got.ranks, ref.ranks)
    with pytest.raises(ValueError):
        sb.tsvdm_tolerance(sb.DenseTensor(a), ts, 0.2, devices=[0, 1])


def test_sharded_pruned_matches_single_gpu(nccl_world1):
    """The certified pruning inside the sharded pipeline (all-reduced slice
    energies, kept slices only through the all-to-all) on c2-like data gives
    the single-GPU result."""
    import torch
    from paper_2605_16058_b200 import configs as cf
    dist = nccl_world1
    a = cf.config2(nlat=46, nlon=90, nt=512, seed=2)
    dims = a.shape
    dev = torch.device("cuda", 0)
    tr = sb.dct_matrix(dims[2])
    ts = sb.TransformSet((tr,))
    ref = sb.tsvdm_tolerance(sb.DenseTensor(a), ts, 1e-2)
    plan = ShardPlan(dims[0], dims[1], dims[2], 1, 0)
    local = torch.from_numpy(scatter_fibres(a, plan).reshape(-1, order="F").copy()).to(dev)
    ops = DeviceOps(tr, dev)
    res = tsvdm_tolerance_sharded(local, plan, ops, 1e-2, dist)
    assert res.pruned > 0
    assert np.array_equal(res.ranks, ref.ranks)
    assert abs(res.discarded_energy - ref.discarded_energy) <= 1e-12 * ref.total_energy
    assert abs(res.total_energy - ref.total_energy) <= 1e-13 * ref.total_energy
    u, g = gather_factors(res, plan, dist)
    assert np.array_equal(u.cpu().numpy(), ref.factors.u_data)
    assert np.array_equal(g.cpu().numpy(), ref.factors.g_data)
    rec = reconstruct_sharded(res, plan, ops, dist)
    err = relative_error_sharded(local, rec, dist, ops=ops)
    assert abs(err - res.relative_error) <= 1e-10 and err <= 1e-2
