"""One ⋆M t-SVDM (tolerance or fixed rank) sharded over ranks (multi-GPU,
one process per GPU).

The reference runs `tsvdm_tolerance` (tsvdm.py:268-321) on one host.  Here
one tensor A (m, p, N) is split over G ranks:

1. Fibre partition.  Column-major A is an (F = m*p) x N matrix whose rows
   are the mode-3 fibres.  Rank g holds fibres [f0_g, f1_g) for every time
   index (``ShardPlan.fibre_bounds``) and applies the transform along time
   to its fibres alone -- the mode-3 product is fibre-local, no exchange.
2. All-to-all.  After the transform rank g's block is (nf_g x N)
   column-major, so the columns (slices) rank h owns, [s0_h, s1_h), are one
   contiguous run: the block is the send buffer as is.  Rank h receives
   nf_g x ns_h values from every g and assembles its ns_h whole slices
   (m*p each) by concatenating the fibre segments in rank order.  This is
   the only data-path collective.
3. Values pass on the owned slices; sigma is all-gathered (r x N, slice
   order) and the global threshold runs replicated on every rank: identical
   inputs give identical ranks, tau and energies, i.e. the reference's
   global semantics (tsvdm.py:85-115).
4. Truncated factors of the owned slices, packed exactly like
   VariableRankFactors restricted to [s0_h, s1_h); concatenating the ranks'
   packed arrays in rank order is the global packed layout.

The compute steps are supplied by an ``ops`` object so the collective logic
is the same for the CUDA path (``DeviceOps``, libstarm kernels) and for the
CPU checks in tests/test_sharded.py (gloo, world size 2).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

__all__ = ["ShardPlan", "ShardedResult", "DeviceOps", "scatter_fibres", "tsvdm_tolerance_sharded",
           "tsvdm_fixed_rank_sharded", "reconstruct_sharded", "relative_error_sharded",
           "gather_factors"]


def _bounds(total: int, world: int, rank: int):
    q, r = divmod(total, world)
    lo = rank * q + min(rank, r)
    return lo, lo + q + (1 if rank < r else 0)


@dataclass(frozen=True)
class ShardPlan:
    m: int
    p: int
    n: int  # number of slices (mode-3 extent)
    world: int
    rank: int

    @property
    def fibres(self) -> int:
        return self.m * self.p

    def fibre_bounds(self, rank=None):
        return _bounds(self.fibres, self.world, self.rank if rank is None else rank)

    def slice_bounds(self, rank=None):
        return _bounds(self.n, self.world, self.rank if rank is None else rank)

    @property
    def nf(self) -> int:
        lo, hi = self.fibre_bounds()
        return hi - lo

    @property
    def ns(self) -> int:
        lo, hi = self.slice_bounds()
        return hi - lo

    def send_counts(self):
        """Elements this rank sends to each rank after the transform."""
        return [self.nf * (b - a) for a, b in (self.slice_bounds(h) for h in range(self.world))]

    def recv_counts(self):
        return [(b - a) * self.ns for a, b in (self.fibre_bounds(g) for g in range(self.world))]


def scatter_fibres(a: np.ndarray, plan: ShardPlan) -> np.ndarray:
    """This rank's fibre block of a column-major (m, p, N) array, as a
    column-major (nf, N) array."""
    f0, f1 = plan.fibre_bounds()
    flat = np.asarray(a).reshape((plan.fibres, plan.n), order="F")
    return np.asfortranarray(flat[f0:f1, :])


def _assemble(recv, plan: ShardPlan, torch):
    """Received fibre segments (grouped by source rank, each nf_g x ns
    column-major) -> ns whole slices, column-major (m*p, ns)."""
    parts = []
    off = 0
    for g in range(plan.world):
        f0, f1 = plan.fibre_bounds(g)
        cnt = (f1 - f0) * plan.ns
        parts.append(recv[off:off + cnt].view(plan.ns, f1 - f0))
        off += cnt
    return torch.cat(parts, dim=1).reshape(-1) if plan.ns else recv[:0]


def _disassemble(slices, plan: ShardPlan, torch):
    """Inverse of _assemble: (m*p, ns) column-major slices -> per-destination
    fibre segments, grouped by rank."""
    if not plan.ns:
        return slices[:0]
    mat = slices.view(plan.ns, plan.fibres)
    parts = []
    for g in range(plan.world):
        f0, f1 = plan.fibre_bounds(g)
        parts.append(mat[:, f0:f1].reshape(-1))
    return torch.cat(parts)


def _all_gather_cols(local, rows, plan: ShardPlan, dist, group, torch):
    """Gather (rows x ns_h) column-major blocks of every rank into
    (rows x N) column-major, slice order."""
    nmax = max(b - a for a, b in (plan.slice_bounds(h) for h in range(plan.world)))
    pad = torch.zeros(rows * nmax, dtype=local.dtype, device=local.device)
    pad[:local.numel()] = local
    out = [torch.empty_like(pad) for _ in range(plan.world)]
    dist.all_gather(out, pad, group=group)
    cols = []
    for h in range(plan.world):
        a, b = plan.slice_bounds(h)
        cols.append(out[h][:rows * (b - a)])
    return torch.cat(cols)


@dataclass
class ShardedResult:
    ranks: np.ndarray          # (N,) int64, identical on every rank
    tau: float
    discarded_energy: float
    total_energy: float
    local_ranks: np.ndarray    # ranks of the owned slices
    u_data: object             # packed factors of the owned slices (torch)
    g_data: object
    slice_ids: np.ndarray = None  # owned slices when not plan.slice_bounds() (pruned path)
    pruned: int = 0               # slices left out by the certified pruning (all ranks)

    @property
    def relative_error(self) -> float:
        return float(np.sqrt(self.discarded_energy / self.total_energy)) if self.total_energy else 0.0


def _owner_ranges(total, world):
    return [_bounds(total, world, h) for h in range(world)]


def _all_gather_var(local, rows, counts, dist, group, torch):
    """All-gather (rows x counts[h]) column-major blocks into (rows x sum)
    in rank order (padded to the largest block for the collective)."""
    world = len(counts)
    nmax = max(max(counts), 1)
    pad = torch.zeros(rows * nmax, dtype=local.dtype, device=local.device)
    pad[:local.numel()] = local
    out = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(out, pad, group=group)
    return torch.cat([out[h][:rows * counts[h]] for h in range(world)])


def _tolerance_pruned_sharded(ahat, plan: ShardPlan, ops, epsilon, dist, group, keep_ids, e0,
                              tbound):
    """The certified slice pruning of compress._tolerance_pruned over the
    ranks.  Every rank chose the same kept slices from all-reduced energies;
    the kept slices are dealt to the ranks in contiguous runs, so the
    all-to-all moves only their fibre segments (c2: 81 of 1024 slices), the
    values pass / threshold (started at e0) / truncated pass run on them, and
    the packed payloads concatenate in rank order to the global layout.
    Returns None when the certificate fails (the caller runs unpruned)."""
    import torch
    m, p, n = plan.m, plan.p, plan.n
    r = min(m, p)
    dev = ahat.device
    world, me = plan.world, plan.rank
    ns_all = int(keep_ids.size)
    own = _owner_ranges(ns_all, world)
    k0, k1 = own[me]
    ns = k1 - k0
    kid = torch.from_numpy(np.ascontiguousarray(keep_ids, dtype=np.int64)).to(dev)
    # (nf x N) column-major = (N, nf) row-major: row t = this rank's fibres of slice t
    send = ahat.view(n, plan.nf).index_select(0, kid).reshape(-1)     # kept rows, in S order
    send_counts = [(b - a) * plan.nf for a, b in own]
    fb = [plan.fibre_bounds(g) for g in range(world)]
    recv_counts = [ns * (f1 - f0) for f0, f1 in fb]
    recv = torch.empty(sum(recv_counts), dtype=torch.float64, device=dev)
    dist.all_to_all_single(recv, send, recv_counts, send_counts, group=group)
    del send
    parts, off = [], 0
    for g in range(world):
        nfg = fb[g][1] - fb[g][0]
        parts.append(recv[off:off + ns * nfg].view(ns, nfg))
        off += ns * nfg
    slices = torch.cat(parts, dim=1).reshape(-1) if ns else recv[:0]
    del recv
    s_local = ops.svd_values(slices, m, p, ns)
    s_all = _all_gather_var(s_local, r, [b - a for a, b in own], dist, group, torch)
    ranks_s, tau, disc, total, cert = ops.threshold_pruned(s_all, r, ns_all, epsilon, e0, tbound)
    if not cert:
        return None
    ranks_s = np.asarray(ranks_s, dtype=np.int64)
    local_ranks = ranks_s[k0:k1].copy()
    u_data, g_data = ops.truncated(slices, m, p, ns, local_ranks, s_local)
    ranks = np.zeros(n, dtype=np.int64)
    ranks[keep_ids] = ranks_s
    return ShardedResult(ranks, float(tau), float(disc), float(total), local_ranks, u_data, g_data,
                         slice_ids=np.asarray(keep_ids[k0:k1], dtype=np.int64),
                         pruned=n - ns_all)


def tsvdm_tolerance_sharded(local, plan: ShardPlan, ops, epsilon, dist, group=None,
                            prune=True) -> ShardedResult:
    """Steps 1-4 of the module docstring.  ``local`` is this rank's (nf, N)
    column-major fibre block as a flat torch tensor on ops' device.  With
    ``prune`` (and ops providing slice_energy / threshold_pruned) the
    certified slice pruning of compress._tolerance_pruned runs first: the
    per-slice energies are this rank's partial sums all-reduced, every rank
    chooses the same slices (compress.prune_choose), and only the kept
    slices cross the all-to-all."""
    import torch
    m, p, n = plan.m, plan.p, plan.n
    r = min(m, p)
    ahat = ops.forward(local, plan.nf, n)                              # 1. transform
    if prune and hasattr(ops, "slice_energy") and hasattr(ops, "threshold_pruned"):
        from .compress import prune_choose
        f = ops.slice_energy(ahat, plan.nf, n)
        dist.all_reduce(f, group=group)
        sel = prune_choose(f.cpu().numpy(), epsilon)
        if sel is not None:
            res = _tolerance_pruned_sharded(ahat, plan, ops, epsilon, dist, group, *sel)
            if res is not None:
                return res
    recv = torch.empty(sum(plan.recv_counts()), dtype=torch.float64, device=ahat.device)
    dist.all_to_all_single(recv, ahat, plan.recv_counts(), plan.send_counts(), group=group)  # 2.
    del ahat
    slices = _assemble(recv, plan, torch)
    del recv
    s_local = ops.svd_values(slices, m, p, plan.ns)                    # 3. values pass
    s_all = _all_gather_cols(s_local, r, plan, dist, group, torch)
    ranks, tau, disc, total = ops.threshold(s_all, r, n, epsilon)     # replicated
    ranks = np.asarray(ranks, dtype=np.int64)
    s0, s1 = plan.slice_bounds()
    local_ranks = ranks[s0:s1].copy()
    u_data, g_data = ops.truncated(slices, m, p, plan.ns, local_ranks, s_local)   # 4.
    return ShardedResult(ranks, float(tau), float(disc), float(total), local_ranks, u_data, g_data)


def tsvdm_fixed_rank_sharded(local, plan: ShardPlan, ops, rank, dist, group=None) -> ShardedResult:
    """Fixed-rank t-SVDM (tsvdm.py:246-265) over the ranks: transform and
    all-to-all as in the tolerance path, then the truncated factors of the
    owned slices WITH their full sigma (keep_values), sigma all-gathered in
    slice order and the tail / total energies (tsvdm.py:260-262) computed
    replicated from the gathered (r x N) matrix -- a fixed summation order,
    so every rank (and every world size) gets the single-GPU numbers."""
    import torch
    m, p, n = plan.m, plan.p, plan.n
    r = min(m, p)
    rank = int(rank)
    if not 1 <= rank <= r:
        raise ValueError(f"rank must lie in [1, {r}], got {rank}")
    ahat = ops.forward(local, plan.nf, n)
    recv = torch.empty(sum(plan.recv_counts()), dtype=torch.float64, device=ahat.device)
    dist.all_to_all_single(recv, ahat, plan.recv_counts(), plan.send_counts(), group=group)
    del ahat
    slices = _assemble(recv, plan, torch)
    del recv
    local_ranks = np.full(plan.ns, rank, dtype=np.int64)
    u_data, g_data, s_local = ops.truncated_with_values(slices, m, p, plan.ns, local_ranks)
    s_all = _all_gather_cols(s_local, r, plan, dist, group, torch)
    disc, total = ops.tail_energy(s_all, r, n, rank)
    ranks = np.full(n, rank, dtype=np.int64)
    return ShardedResult(ranks, 0.0, float(disc), float(total), local_ranks, u_data, g_data)


def reconstruct_sharded(res: ShardedResult, plan: ShardPlan, ops, dist, group=None):
    """This rank's fibre block of the reconstruction (flat (nf, N) col-major):
    facewise U_i G_i of the owned slices, all-to-all back to fibres, inverse
    transform.  Pruned results own a subset of the slices (res.slice_ids);
    the other slices are zero."""
    import torch
    if res.slice_ids is not None:
        return _reconstruct_pruned(res, plan, ops, dist, group)
    chat = ops.unpack(res.u_data, res.g_data, res.local_ranks, plan.m, plan.p, plan.ns)
    send = _disassemble(chat, plan, torch)
    del chat
    back = torch.empty(plan.nf * plan.n, dtype=torch.float64, device=send.device)
    # roles swap: send ns x nf_g to g, receive nf x ns_h from h
    dist.all_to_all_single(back, send, plan.send_counts(), plan.recv_counts(), group=group)
    del send
    return ops.inverse(back, plan.nf, plan.n)


def _reconstruct_pruned(res: ShardedResult, plan: ShardPlan, ops, dist, group):
    import torch
    world = plan.world
    ids = torch.from_numpy(np.ascontiguousarray(res.slice_ids, dtype=np.int64))
    ns = int(ids.numel())
    counts = torch.tensor([ns], dtype=torch.int64)
    dev = getattr(ops, "device", None)
    if dev is not None:
        counts = counts.to(dev)
    allc = [torch.empty_like(counts) for _ in range(world)]
    dist.all_gather(allc, counts, group=group)
    allc = [int(c.item()) for c in allc]
    # every rank's slice ids, in rank order
    idt = ids.to(dev) if dev is not None else ids
    all_ids = _all_gather_var(idt.to(torch.float64), 1, allc, dist, group, torch).to(torch.int64)
    chat = ops.unpack(res.u_data, res.g_data, res.local_ranks, plan.m, plan.p, ns)
    fb = [plan.fibre_bounds(g) for g in range(world)]
    mat = chat.view(ns, plan.fibres) if ns else chat.view(0, plan.fibres)
    send = torch.cat([mat[:, a:b].reshape(-1) for a, b in fb]) if ns else chat[:0]
    send_counts = [ns * (b - a) for a, b in fb]
    recv_counts = [allc[h] * plan.nf for h in range(world)]
    recv = torch.empty(sum(recv_counts), dtype=torch.float64, device=chat.device)
    dist.all_to_all_single(recv, send, recv_counts, send_counts, group=group)
    back = torch.zeros(plan.n, plan.nf, dtype=torch.float64, device=chat.device)
    if all_ids.numel():
        back.index_copy_(0, all_ids.to(back.device), recv.view(-1, plan.nf))
    return ops.inverse(back.reshape(-1), plan.nf, plan.n)


def relative_error_sharded(local, rec, dist, group=None, ops=None) -> float:
    """||A - rec|| / ||A|| over all ranks: per-rank (sum (a-b)^2, sum a^2)
    by ``ops.error_sums`` (the K10 kernel on the device) and one all-reduce
    of the two partials."""
    import torch
    if ops is not None and hasattr(ops, "error_sums"):
        sums = ops.error_sums(local, rec)
    else:
        sums = torch.stack([torch.sum((local - rec) ** 2), torch.sum(local ** 2)]).to(torch.float64)
    dist.all_reduce(sums, group=group)
    num, den = (float(v) for v in sums.cpu())
    return float(np.sqrt(num / den)) if den else 0.0


def gather_factors(res: ShardedResult, plan: ShardPlan, dist, group=None):
    """Concatenate the ranks' packed factors (global packed layout) on every
    rank: (u_data, g_data) torch tensors."""
    import torch
    out = []
    for data in (res.u_data, res.g_data):
        n_local = torch.tensor([data.numel()], dtype=torch.int64, device=data.device)
        sizes = [torch.empty_like(n_local) for _ in range(plan.world)]
        dist.all_gather(sizes, n_local, group=group)
        sizes = [int(s.item()) for s in sizes]
        pad = torch.zeros(max(max(sizes), 1), dtype=data.dtype, device=data.device)
        pad[:data.numel()] = data
        parts = [torch.empty_like(pad) for _ in range(plan.world)]
        dist.all_gather(parts, pad, group=group)
        out.append(torch.cat([parts[h][:sizes[h]] for h in range(plan.world)]))
    return tuple(out)


class DeviceOps:
    """The CUDA (libstarm) implementation of the per-rank compute steps."""

    def __init__(self, transform, device):
        from .transform_set import TransformSet
        self.ts = TransformSet((transform,))
        self.device = device

    def _dev(self, flat, dims):
        from .tensors import DeviceTensor
        return DeviceTensor(flat, dims)

    def forward(self, flat, nf, n):
        from .mode_product import forward_device
        return forward_device(self._dev(flat, (nf, 1, n)), self.ts).data

    def inverse(self, flat, nf, n):
        from .mode_product import inverse_device
        return inverse_device(self._dev(flat, (nf, 1, n)), self.ts).data

    def svd_values(self, slices, m, p, ns):
        """Values pass of the owned slices; keeps each slice's factorisation
        state (when it fits in HBM) so the following truncated pass on the
        same slices does not refactor them (tsvdm_tolerance's schedule)."""
        import torch
        from .compress import _state_fits
        from .slice_svd import svd_values_device
        self._state = None
        if ns == 0:
            return torch.empty(0, dtype=torch.float64, device=self.device)
        x = self._dev(slices, (m, p, ns))
        if _state_fits(x):
            s, state = svd_values_device(x, keep_state=True)
            self._state = (slices.data_ptr(), ns, state) if state is not None else None
            return s
        return svd_values_device(x)

    def threshold(self, s_all, r, n, epsilon):
        from .compress import threshold_device
        ranks, scal, _, _, _ = threshold_device(s_all, r, n, epsilon)
        sc = scal.cpu().numpy()
        return ranks.cpu().numpy(), sc[0], sc[1], sc[2]

    def truncated(self, slices, m, p, ns, local_ranks, s_local):
        import torch
        from .slice_svd import svd_truncated_device
        total = int(np.sum(local_ranks))
        if ns == 0 or total == 0:
            z = torch.empty(0, dtype=torch.float64, device=self.device)
            return z, z
        rk = torch.from_numpy(np.ascontiguousarray(local_ranks)).to(self.device)
        st = getattr(self, "_state", None)
        state = st[2] if st is not None and st[0] == slices.data_ptr() and st[1] == ns else None
        f, _ = svd_truncated_device(self._dev(slices, (m, p, ns)), rk, total, state=state)
        self._state = None
        return f.u_data[:total * m], f.g_data[:total * p]

    def truncated_with_values(self, slices, m, p, ns, local_ranks):
        """Packed leading factors AND every sigma of the owned slices (the
        keep_values pass of tsvdm_fixed_rank): (u_data, g_data, s (r*ns))."""
        import torch
        from .slice_svd import svd_truncated_device
        r = min(m, p)
        total = int(np.sum(local_ranks))
        if ns == 0:
            z = torch.empty(0, dtype=torch.float64, device=self.device)
            return z, z, z
        rk = torch.from_numpy(np.ascontiguousarray(local_ranks)).to(self.device)
        f, s = svd_truncated_device(self._dev(slices, (m, p, ns)), rk, total, keep_values=True)
        return f.u_data[:total * m], f.g_data[:total * p], s[:r * ns]

    def slice_energy(self, ahat, nf, n):
        """Per-slice energies of this rank's fibres: column sums of squares of
        the (nf x N) column-major block (starm_slice_energy_f64)."""
        import torch
        from . import _native as nat
        f = torch.empty(n, dtype=torch.float64, device=self.device)
        nat.call("starm_slice_energy_f64", ahat.data_ptr(), nf, n, f.data_ptr(),
                 nat.stream_ptr(self.device))
        return f

    def threshold_pruned(self, s_all, r, n, epsilon, e0, tbound):
        import torch
        from . import _native as nat
        lib = nat.load()
        nbytes = lib.starm_threshold_workspace_bytes(r, n)
        ws = nat.workspace(nbytes, self.device)
        ranks = torch.empty(n, dtype=torch.int64, device=self.device)
        scal = torch.empty(3, dtype=torch.float64, device=self.device)
        j = torch.empty(1, dtype=torch.int64, device=self.device)
        cert = torch.empty(1, dtype=torch.int32, device=self.device)
        nat.call("starm_threshold_pruned_f64", s_all.data_ptr(), r, n, float(epsilon), float(e0),
                 float(tbound), ranks.data_ptr(), scal.data_ptr(), j.data_ptr(), cert.data_ptr(),
                 ws.data_ptr(), nbytes, nat.stream_ptr(self.device))
        sc = scal.cpu().numpy()
        return ranks.cpu().numpy(), sc[0], sc[1], sc[2], bool(cert.item())

    def tail_energy(self, s_all, r, n, rank):
        import torch
        from . import _native as nat
        en = torch.empty(2, dtype=torch.float64, device=self.device)
        nat.call("starm_tail_energy_f64", s_all.data_ptr(), r, n, int(rank), en.data_ptr(),
                 nat.stream_ptr(self.device))
        d, t = en.cpu().numpy()
        return float(d), float(t)

    def error_sums(self, a, b):
        """(sum (a-b)^2, sum a^2) of two flat device tensors (K10)."""
        import torch
        from . import _native as nat
        lib = nat.load()
        out = torch.zeros(2, dtype=torch.float64, device=self.device)
        if a.numel() == 0:
            return out
        nbytes = lib.starm_error_sums_workspace_bytes(a.numel())
        ws = nat.workspace(nbytes, self.device)
        nat.call("starm_error_sums_f64", a.data_ptr(), b.data_ptr(), a.numel(), out.data_ptr(),
                 ws.data_ptr(), nbytes, nat.stream_ptr(self.device))
        return out

    def unpack(self, u_data, g_data, local_ranks, m, p, ns):
        import torch
        from . import _native as nat
        out = torch.empty(m * p * ns, dtype=torch.float64, device=self.device)
        if ns == 0:
            return out
        rk = torch.from_numpy(np.ascontiguousarray(local_ranks)).to(self.device)
        u_off = torch.empty(ns + 1, dtype=torch.int64, device=self.device)
        g_off = torch.empty(ns + 1, dtype=torch.int64, device=self.device)
        st = nat.stream_ptr(self.device)
        nat.call("starm_pack_offsets", rk.data_ptr(), ns, m, p, u_off.data_ptr(), g_off.data_ptr(), st)
        u = u_data if u_data.numel() else torch.zeros(1, dtype=torch.float64, device=self.device)
        g = g_data if g_data.numel() else torch.zeros(1, dtype=torch.float64, device=self.device)
        nat.call("starm_unpack_facewise_f64", u.data_ptr(), g.data_ptr(), rk.data_ptr(),
                 u_off.data_ptr(), g_off.data_ptr(), m, p, ns, out.data_ptr(), st)
        return out
