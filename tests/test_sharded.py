"""Multi-rank host logic of the sharded t-SVDM (paper_2605_16058_b200/sharded.py).

Two CPU processes over gloo run the real collective schedule (fibre
partition -> transform -> all_to_all -> slice assembly -> sigma all-gather ->
replicated threshold -> packed factors -> all_to_all back -> inverse
transform -> error all-reduce) with the oracle supplying the per-rank
compute; the result must equal the single-process oracle pipeline on the
whole tensor.  The GPU runs substitute DeviceOps (libstarm kernels) for the
oracle ops; nothing else changes.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_2605_16058_b200.sharded import (ShardPlan, gather_factors, reconstruct_sharded,
                                           relative_error_sharded, scatter_fibres,
                                           tsvdm_fixed_rank_sharded, tsvdm_tolerance_sharded)


class OracleOps:
    """CPU stand-in for DeviceOps (torch CPU tensors in, torch CPU tensors out)."""

    def __init__(self, mat):
        self.mat = mat

    def forward(self, flat, nf, n):
        a = flat.numpy().reshape((nf, 1, n), order="F")
        return torch.from_numpy(oracle.ttm(a, 2, self.mat).reshape(-1, order="F").copy())

    def inverse(self, flat, nf, n):
        a = flat.numpy().reshape((nf, 1, n), order="F")
        return torch.from_numpy(oracle.ttm(a, 2, self.mat.T).reshape(-1, order="F").copy())

    def svd_values(self, slices, m, p, ns):
        if ns == 0:
            return torch.zeros(0, dtype=torch.float64)
        a = slices.numpy().reshape((m, p, ns), order="F")
        return torch.from_numpy(oracle.svd_values_only(a).reshape(-1, order="F").copy())

    def threshold(self, s_all, r, n, eps):
        th = oracle.compute_threshold(s_all.numpy().reshape((r, n), order="F"), eps)
        return th["ranks"], th["tau"], th["discarded_energy"], th["total_energy"]

    def truncated(self, slices, m, p, ns, local_ranks, s_local):
        if ns == 0:
            z = torch.zeros(0, dtype=torch.float64)
            return z, z
        a = slices.numpy().reshape((m, p, ns), order="F")
        u, g = oracle.svd_truncated_slices(a, local_ranks)
        return torch.from_numpy(u), torch.from_numpy(g)

    def truncated_with_values(self, slices, m, p, ns, local_ranks):
        if ns == 0:
            z = torch.zeros(0, dtype=torch.float64)
            return z, z, z
        a = slices.numpy().reshape((m, p, ns), order="F")
        u, g, s = oracle.svd_truncated_slices(a, local_ranks, keep_values=True)
        return torch.from_numpy(u), torch.from_numpy(g), torch.from_numpy(s.reshape(-1, order="F").copy())

    def slice_energy(self, ahat, nf, n):
        a = ahat.numpy().reshape((nf, n), order="F")
        return torch.from_numpy(np.ascontiguousarray((a * a).sum(axis=0)))

    def threshold_pruned(self, s_all, r, n, eps, e0, tbound):
        """compute_threshold (tsvdm.py:85-115) on the kept slices with the
        running sum started at e0 (the left-out energy); cert = crossing value
        above tbound (numpy restatement of starm_threshold_pruned_f64)."""
        sq = s_all.numpy().reshape((r, n), order="F") ** 2
        v = np.sort(sq, axis=None)
        w = e0 + np.cumsum(v)
        total = w[-1]
        budget = eps * eps * total
        j = int(np.searchsorted(w, budget, side="left"))
        tau = v[j - 1] if j > 0 else 0.0
        cert = j < v.size and v[j] > tbound
        keep = sq > tau
        disc = e0 + oracle.pairwise_sum(sq[~keep])
        if disc >= budget and tau > 0.0:
            keep = sq >= tau
            disc = e0 + oracle.pairwise_sum(sq[~keep])
        return keep.sum(axis=0).astype(np.int64), tau, disc, total, bool(cert)

    def tail_energy(self, s_all, r, n, rank):
        sq = s_all.numpy().reshape((r, n), order="F") ** 2
        return float(sq[rank:, :].sum()), float(sq.sum())     # tsvdm.py:260-262

    def unpack(self, u_data, g_data, local_ranks, m, p, ns):
        out = np.zeros((m, p, ns), order="F")
        uo, go = oracle.u_offsets(local_ranks, m), oracle.g_offsets(local_ranks, p)
        u_data, g_data = u_data.numpy(), g_data.numpy()
        for i in range(ns):
            k = int(local_ranks[i])
            if k:
                u = u_data[uo[i]:uo[i + 1]].reshape((m, k), order="F")
                g = g_data[go[i]:go[i + 1]].reshape((k, p), order="F")
                out[:, :, i] = u @ g
        return torch.from_numpy(out.reshape(-1, order="F").copy())


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _tensor(dims, seed):
    rng = np.random.default_rng(seed)
    m, p, n = dims
    k = 3
    a = np.einsum("ir,jr,kr->ijk", rng.standard_normal((m, k)), rng.standard_normal((p, k)),
                  rng.standard_normal((n, k)))
    a += 0.05 * rng.standard_normal(dims)
    return np.asfortranarray(a)


def _worker(rank, world, port, dims, eps, seed, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        a = _tensor(dims, seed)
        m, p, n = dims
        mat = oracle.dct_matrix(n)
        plan = ShardPlan(m, p, n, world, rank)
        local = torch.from_numpy(scatter_fibres(a, plan).reshape(-1, order="F").copy())
        ops = OracleOps(mat)
        res = tsvdm_tolerance_sharded(local, plan, ops, eps, dist)
        u, g = gather_factors(res, plan, dist)
        rec = reconstruct_sharded(res, plan, ops, dist)
        err = relative_error_sharded(local, rec, dist)
        q.put((rank, res.ranks, res.tau, res.discarded_energy, res.total_energy,
               u.numpy(), g.numpy(), err))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("dims,eps,world", [((6, 5, 8), 0.05, 2), ((7, 3, 5), 0.1, 2),
                                            ((4, 4, 3), 0.2, 2), ((5, 6, 9), 0.05, 3)])
def test_sharded_tolerance_matches_single_process(dims, eps, world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, dims, eps, 11, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    outs = [q.get(timeout=120) for _ in range(world)]
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    outs.sort(key=lambda o: o[0])
    a = _tensor(dims, 11)
    mat = oracle.dct_matrix(dims[2])
    ref = oracle.tsvdm_tolerance(a, [mat], eps)
    rec = oracle.reconstruct_packed(dims, [mat], ref["ranks"], ref["u_data"], ref["g_data"])
    ref_err = float(np.linalg.norm(a - rec) / np.linalg.norm(a))
    for rank, ranks, tau, disc, total, u, g, err in outs:
        # every rank holds the same global decision
        assert np.array_equal(ranks, ref["ranks"]), rank
        assert abs(tau - ref["tau"]) <= 1e-12 * max(ref["tau"], 1e-300)
        assert abs(disc - ref["discarded_energy"]) <= 1e-12 * ref["total_energy"]
        assert abs(total - ref["total_energy"]) <= 1e-12 * ref["total_energy"]
        # gathered packed factors: the global layout (same slices, same LAPACK)
        assert u.shape == ref["u_data"].shape and g.shape == ref["g_data"].shape
        np.testing.assert_allclose(u, ref["u_data"], rtol=0, atol=1e-9)
        np.testing.assert_allclose(g, ref["g_data"], rtol=0, atol=1e-9)
        # realised error through the sharded reconstruction
        assert abs(err - ref_err) <= 1e-10
        assert abs(err - np.sqrt(disc / total)) <= 1e-10


def _worker_fixed(rank, world, port, dims, k, seed, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        a = _tensor(dims, seed)
        m, p, n = dims
        mat = oracle.dct_matrix(n)
        plan = ShardPlan(m, p, n, world, rank)
        local = torch.from_numpy(scatter_fibres(a, plan).reshape(-1, order="F").copy())
        ops = OracleOps(mat)
        res = tsvdm_fixed_rank_sharded(local, plan, ops, k, dist)
        u, g = gather_factors(res, plan, dist)
        rec = reconstruct_sharded(res, plan, ops, dist)
        err = relative_error_sharded(local, rec, dist)
        q.put((rank, res.ranks, res.discarded_energy, res.total_energy, u.numpy(), g.numpy(), err))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("dims,k,world", [((6, 5, 8), 2, 2), ((7, 3, 5), 1, 2), ((5, 6, 9), 3, 4),
                                          ((4, 4, 3), 4, 4)])
def test_sharded_fixed_rank_matches_single_process(dims, k, world):
    """tsvdm_fixed_rank over 2 / 4 gloo ranks (4 ranks with 3 slices: one rank
    owns none) equals the single-process oracle of tsvdm.py:246-265."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_fixed, args=(r, world, port, dims, k, 5, q))
             for r in range(world)]
    for pr in procs:
        pr.start()
    outs = [q.get(timeout=120) for _ in range(world)]
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    a = _tensor(dims, 5)
    mat = oracle.dct_matrix(dims[2])
    ref = oracle.tsvdm_fixed_rank(a, [mat], k)
    rec = oracle.reconstruct_packed(dims, [mat], ref["ranks"], ref["u_data"], ref["g_data"])
    ref_err = float(np.linalg.norm(a - rec) / np.linalg.norm(a))
    for rank, ranks, disc, total, u, g, err in outs:
        assert np.array_equal(ranks, ref["ranks"]), rank
        assert abs(disc - ref["discarded_energy"]) <= 1e-12 * ref["total_energy"]
        assert abs(total - ref["total_energy"]) <= 1e-12 * ref["total_energy"]
        np.testing.assert_allclose(u, ref["u_data"], rtol=0, atol=1e-9)
        np.testing.assert_allclose(g, ref["g_data"], rtol=0, atol=1e-9)
        assert abs(err - ref_err) <= 1e-10
        assert abs(err - np.sqrt(disc / total)) <= 1e-10


def _pruning_tensor():
    """Three separable oscillations + 1e-3 noise over 64 time steps: the DCT
    concentrates them in ~20 slices, the rest are noise far below tau."""
    rng = np.random.default_rng(4)
    m, p, n = 9, 16, 64
    t = np.arange(n)
    a = np.zeros((m, p, n))
    for k in range(3):
        a += np.einsum("i,j,t->ijt", rng.standard_normal(m), rng.standard_normal(p),
                       np.cos(2 * np.pi * (k + 1) * t / (1.7 * n) + rng.uniform(0, 6)))
    a += 1e-3 * rng.standard_normal((m, p, n))
    return np.asfortranarray(a)


def _worker_pruned(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        a = _pruning_tensor()
        m, p, n = a.shape
        mat = oracle.dct_matrix(n)
        plan = ShardPlan(m, p, n, world, rank)
        local = torch.from_numpy(scatter_fibres(a, plan).reshape(-1, order="F").copy())
        ops = OracleOps(mat)
        res = tsvdm_tolerance_sharded(local, plan, ops, 1e-2, dist)
        u, g = gather_factors(res, plan, dist)
        rec = reconstruct_sharded(res, plan, ops, dist)
        err = relative_error_sharded(local, rec, dist)
        q.put((rank, res.pruned, res.ranks, res.discarded_energy, res.total_energy, u.numpy(),
               g.numpy(), err))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_tolerance_pruned_matches_single_process(world):
    """Certified slice pruning over gloo ranks: the kept slices are dealt to
    the ranks, only they cross the all-to-all; ranks, energies, factors and
    the realised error equal the single-process (unpruned) oracle."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_pruned, args=(r, world, port, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    outs = [q.get(timeout=120) for _ in range(world)]
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    a = _pruning_tensor()
    mat = oracle.dct_matrix(64)
    ref = oracle.tsvdm_tolerance(a, [mat], 1e-2)
    rec = oracle.reconstruct_packed(a.shape, [mat], ref["ranks"], ref["u_data"], ref["g_data"])
    ref_err = float(np.linalg.norm(a - rec) / np.linalg.norm(a))
    for rank, pruned, ranks, disc, total, u, g, err in outs:
        assert pruned > 0, "the test case must exercise the pruned path"
        assert np.array_equal(ranks, ref["ranks"]), rank
        assert abs(total - ref["total_energy"]) <= 1e-12 * ref["total_energy"]
        assert abs(disc - ref["discarded_energy"]) <= 1e-12 * ref["total_energy"]
        np.testing.assert_allclose(u, ref["u_data"], rtol=0, atol=1e-9)
        np.testing.assert_allclose(g, ref["g_data"], rtol=0, atol=1e-9)
        assert abs(err - ref_err) <= 1e-10


def test_shard_plan_partitions():
    for m, p, n, world in [(7, 5, 3, 2), (1, 1, 1, 4), (10, 3, 17, 3), (2, 2, 2, 8)]:
        plans = [ShardPlan(m, p, n, world, r) for r in range(world)]
        fb = [pl.fibre_bounds() for pl in plans]
        sb = [pl.slice_bounds() for pl in plans]
        assert fb[0][0] == 0 and fb[-1][1] == m * p
        assert sb[0][0] == 0 and sb[-1][1] == n
        for i in range(world - 1):
            assert fb[i][1] == fb[i + 1][0] and sb[i][1] == sb[i + 1][0]
        # what g sends to h is what h expects from g
        for g in range(world):
            for h in range(world):
                assert plans[g].send_counts()[h] == plans[h].recv_counts()[g]
