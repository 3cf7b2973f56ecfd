"""numpy/scipy restatement of the reference t-SVDM hot path (TEST ORACLE).

TEST INFRASTRUCTURE ONLY -- see ``oracle/__init__.py``.  Every function
cites the reference file:line it restates (paths relative to
``/root/reference/pkg/src/starm/``).  Arrays are plain numpy float64 arrays
in column-major (Fortran) order, exactly the storage of the reference's
``DenseTensor`` (tensor.py:76-98).

Third-party arithmetic: like the reference, the per-slice SVD is LAPACK
``dgesvd`` reached through ``scipy.linalg.get_lapack_funcs`` (scipy 1.18.1
bundling OpenBLAS 0.3.30 in this image) and the contractions are
``np.matmul`` (numpy 2.3.5 / OpenBLAS DGEMM).  The reference pins only lower
bounds (pyproject.toml:12-16: numpy>=1.24, scipy>=1.10).
"""

from __future__ import annotations

import math
from math import prod

import numpy as np
from scipy.linalg import get_lapack_funcs
from threadpoolctl import threadpool_limits

__all__ = [
    "dct_matrix", "orthonormality_residual", "ttm", "to_transform_domain",
    "from_transform_domain", "slice_svd", "svd_all_slices", "svd_values_only",
    "svd_truncated_slices", "pairwise_sum", "sequential_cumsum",
    "compute_threshold", "tsvdm_fixed_rank", "tsvdm_tolerance",
    "reconstruct_packed", "starm_product", "full_tsvdm_reconstruct",
    "u_offsets", "g_offsets",
]

_gesvd, _gesvd_lwork = get_lapack_funcs(
    ("gesvd", "gesvd_lwork"), (np.empty(0, dtype=np.float64),)
)


# ---------------------------------------------------------------- transforms

def dct_matrix(n: int) -> np.ndarray:
    """Orthonormal DCT-II, transforms.py:77-91."""
    j = np.arange(n)[:, None]
    k = np.arange(n)[None, :]
    mat = np.cos(np.pi * (2 * k + 1) * j / (2.0 * n))
    mat[0, :] *= np.sqrt(1.0 / n)
    if n > 1:
        mat[1:, :] *= np.sqrt(2.0 / n)
    return np.asfortranarray(mat)


def orthonormality_residual(m) -> float:
    """``||M^T M - I||_F / sqrt(n)``, transforms.py:22-27."""
    m = np.asarray(m, dtype=np.float64)
    g = m.T @ m
    g[np.diag_indices(g.shape[0])] -= 1.0
    return float(np.linalg.norm(g) / np.sqrt(g.shape[0]))


# ----------------------------------------------------------------------- TTM

def ttm(arr: np.ndarray, mode: int, mat: np.ndarray, threads: int = 1) -> np.ndarray:
    """Mode-``mode`` product, ttm.py:87-104 with the batched dispatch of
    ttm.py:113-122: the column-major buffer viewed C-order as
    (batch, inner, rows) and ``dst[b] = mat @ src[b]``."""
    dims = arr.shape
    mat = np.asarray(mat, dtype=np.float64)
    rows = prod(dims[:mode])
    inner = dims[mode]
    batch = prod(dims[mode + 1:])
    assert mat.shape[1] == inner
    flat = arr.reshape(-1, order="F")
    src = flat.reshape(batch, inner, rows)
    out = np.empty(batch * mat.shape[0] * rows)
    # reference default threads=1 (ttm.py:87,121): same BLAS blocking -> same bits
    with threadpool_limits(limits=threads, user_api="blas"):
        np.matmul(mat, src, out=out.reshape(batch, mat.shape[0], rows))
    out_dims = dims[:mode] + (mat.shape[0],) + dims[mode + 1:]
    return out.reshape(out_dims, order="F")


def to_transform_domain(arr, mats):
    """Ascending modes, ttm.py:138-144."""
    out = arr
    for k, m in enumerate(mats, start=2):
        out = ttm(out, k, m)
    return out


def from_transform_domain(arr, mats, inverses=None):
    """Descending modes with M^T, ttm.py:147-153 (ttm_inverse = transpose,
    ttm.py:107-110).  ``inverses`` lets the config-4 restatement (SURVEY
    §8c) substitute explicit M^-1 matrices for the transposes."""
    out = arr
    for k in range(len(mats) + 1, 1, -1):
        mk = mats[k - 2].T if inverses is None else inverses[k - 2]
        out = ttm(out, k, mk)
    return out


# ----------------------------------------------------------------- slice SVD

def slice_svd(mat: np.ndarray, index: int = 0):
    """Thin SVD of one slice, slicesvd.py:42-62 (LAPACK dgesvd jobu=jobvt=S,
    zero-slice identity bases, non-finite ValueError naming the slice)."""
    if not np.isfinite(mat).all():
        raise ValueError(f"slice {index} contains non-finite values")
    m, p = mat.shape
    r = min(m, p)
    if not mat.any():
        return np.eye(m, r, order="F"), np.zeros(r), np.eye(r, p, order="F")
    lwork, info = _gesvd_lwork(m, p, compute_uv=1, full_matrices=0)
    scratch = np.array(mat, order="F", copy=True)
    u, s, vt, info = _gesvd(scratch, compute_uv=1, full_matrices=0,
                            lwork=int(lwork), overwrite_a=1)
    if info != 0:
        raise np.linalg.LinAlgError(f"SVD did not converge on slice {index} (info={info})")
    return u, s, vt


def _slices(arr):
    m, p = arr.shape[0], arr.shape[1]
    n = prod(arr.shape[2:])
    return arr.reshape((m, p, n), order="F")


def svd_all_slices(arr, indices=None):
    """slicesvd.py:115-136: U (m,r,N), s (r,N), V (p,r,N).  ``indices``
    restricts the work to a subset of slices (for bounded CPU samples)."""
    sl = _slices(arr)
    m, p, n = sl.shape
    r = min(m, p)
    idx = range(n) if indices is None else indices
    u_out = np.zeros((m, r, n), order="F")
    s_out = np.zeros((r, n), order="F")
    v_out = np.zeros((p, r, n), order="F")
    for i in idx:
        u, s, vt = slice_svd(sl[:, :, i], i)
        u_out[:, :, i] = u
        s_out[:, i] = s
        v_out[:, :, i] = vt.T
    return u_out, s_out, v_out


def svd_values_only(arr, indices=None):
    """slicesvd.py:139-177 (values of the same dgesvd call)."""
    sl = _slices(arr)
    m, p, n = sl.shape
    idx = range(n) if indices is None else indices
    s_out = np.zeros((min(m, p), n), order="F")
    for i in idx:
        s_out[:, i] = slice_svd(sl[:, :, i], i)[1]
    return s_out


def u_offsets(ranks, m):
    off = np.zeros(len(ranks) + 1, dtype=np.int64)
    np.cumsum(np.asarray(ranks, dtype=np.int64) * m, out=off[1:])
    return off


def g_offsets(ranks, p):
    return u_offsets(ranks, p)


def svd_truncated_slices(arr, ranks, keep_values=False):
    """slicesvd.py:259-292: packed ``u_data`` (m x k blocks, col-major) and
    ``g_data`` (k x p blocks of diag(s) V^T) in slice order, offsets from
    slicesvd.py:208-211.  Rank-zero slices skipped unless keep_values."""
    sl = _slices(arr)
    m, p, n = sl.shape
    ranks = np.asarray(ranks, dtype=np.int64)
    uo, go = u_offsets(ranks, m), g_offsets(ranks, p)
    u_data = np.empty(int(uo[-1]))
    g_data = np.empty(int(go[-1]))
    values = np.empty((min(m, p), n), order="F") if keep_values else None
    for i in range(n):
        k = int(ranks[i])
        if k == 0 and values is None:
            continue
        u, s, vt = slice_svd(sl[:, :, i], i)
        if values is not None:
            values[:, i] = s
        if k:
            u_data[uo[i]:uo[i + 1]] = u[:, :k].reshape(-1, order="F")
            g_data[go[i]:go[i + 1]] = (s[:k, None] * vt[:k, :]).reshape(-1, order="F")
    return (u_data, g_data, values) if keep_values else (u_data, g_data)


# ----------------------------------------------------------------- threshold

def pairwise_sum(a) -> float:
    """numpy's float64 add-reduce of a contiguous 1-D array: a zero start plus
    the pairwise tree of numpy/_core/src/umath/loops_utils.h.src (blocks of
    <=128 with 8 accumulators, halving split rounded down to a multiple of
    8).  Verified bit-identical to ``np.sum`` in tests/test_oracle_golden.py.
    This is the summation order ``compute_threshold`` inherits from
    ``squared[~keep].sum()`` (tsvdm.py:108,112)."""
    a = np.ascontiguousarray(a, dtype=np.float64)

    def rec(lo, n):
        if n < 8:
            res = -0.0
            for i in range(lo, lo + n):
                res += a[i]
            return res
        if n <= 128:
            r = [float(a[lo + j]) for j in range(8)]
            i = 8
            stop = n - (n % 8)
            while i < stop:
                for j in range(8):
                    r[j] += a[lo + i + j]
                i += 8
            res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]))
            while i < n:
                res += a[lo + i]
                i += 1
            return res
        n2 = n // 2
        n2 -= n2 % 8
        return rec(lo, n2) + rec(lo + n2, n - n2)

    return float(0.0 + rec(0, a.size)) if a.size else 0.0


def sequential_cumsum(v) -> np.ndarray:
    """Left-to-right running sums (``np.cumsum`` of a 1-D float64 array is
    sequential)."""
    return np.cumsum(np.asarray(v, dtype=np.float64))


def compute_threshold(s, epsilon):
    """tsvdm.py:85-115, returned as a dict of the ThresholdResult fields."""
    epsilon = float(epsilon)
    if not 0.0 < epsilon < 1.0:
        raise ValueError(f"tolerance must lie in (0, 1), got {epsilon}")
    s = np.asarray(s, dtype=np.float64)
    squared = s * s
    v = np.sort(squared, axis=None)
    w = np.cumsum(v)
    total = float(w[-1]) if w.size else 0.0
    if total == 0.0:
        return dict(v=v, w=w, j=0, tau=0.0,
                    ranks=np.zeros(s.shape[1], dtype=np.int64),
                    discarded_energy=0.0, total_energy=0.0)
    budget = epsilon * epsilon * total
    j = int(np.searchsorted(w, budget, side="left"))
    tau = float(v[j - 1]) if j > 0 else 0.0
    keep = squared > tau
    discarded = float(squared[~keep].sum())
    if discarded >= budget and tau > 0.0:
        keep = squared >= tau
        discarded = float(squared[~keep].sum())
    ranks = keep.sum(axis=0).astype(np.int64)
    return dict(v=v, w=w, j=j, tau=tau, ranks=ranks,
                discarded_energy=discarded, total_energy=total)


# ---------------------------------------------------------------- pipelines

def tsvdm_fixed_rank(arr, mats, rank):
    """tsvdm.py:246-265 (TTM -> svd_truncated_slices(keep_values) -> tail
    and total energies)."""
    ahat = to_transform_domain(arr, mats)
    n = prod(arr.shape[2:])
    ranks = np.full(n, int(rank), dtype=np.int64)
    u_data, g_data, values = svd_truncated_slices(ahat, ranks, keep_values=True)
    sq = values * values
    return dict(ranks=ranks, u_data=u_data, g_data=g_data, s=values,
                discarded_energy=float(sq[rank:, :].sum()),
                total_energy=float(sq.sum()))


def tsvdm_tolerance(arr, mats, epsilon, ahat=None):
    """tsvdm.py:268-321, memory-efficient strategy (values pass, threshold,
    second factorization of the slices with rank > 0)."""
    if ahat is None:
        ahat = to_transform_domain(arr, mats)
    values = svd_values_only(ahat)
    th = compute_threshold(values, epsilon)
    u_data, g_data = svd_truncated_slices(ahat, th["ranks"])
    out = dict(th)
    out.update(s=values, u_data=u_data, g_data=g_data)
    return out


def reconstruct_packed(dims, mats, ranks, u_data, g_data, inverses=None):
    """tsvdm.py:342-357: zero-filled facewise U_i G_i, then the inverse
    transforms in descending mode order."""
    m, p = dims[0], dims[1]
    n = prod(dims[2:])
    ranks = np.asarray(ranks, dtype=np.int64)
    uo, go = u_offsets(ranks, m), g_offsets(ranks, p)
    chat = np.zeros((m, p, n), order="F")
    for i in range(n):
        k = int(ranks[i])
        if k:
            u = u_data[uo[i]:uo[i + 1]].reshape((m, k), order="F")
            g = g_data[go[i]:go[i + 1]].reshape((k, p), order="F")
            chat[:, :, i] = u @ g
    return from_transform_domain(chat.reshape(dims, order="F"), mats, inverses)


def starm_product(a, b, mats):
    """tsvdm.py:219-233 with _facewise_matmul (tsvdm.py:205-216)."""
    ahat = to_transform_domain(a, mats)
    bhat = to_transform_domain(b, mats)
    m, p = a.shape[0], a.shape[1]
    cols = b.shape[1]
    n = prod(a.shape[2:])
    a_c = ahat.reshape(-1, order="F").reshape(n, p, m)
    b_c = bhat.reshape(-1, order="F").reshape(n, cols, p)
    out = np.empty(m * cols * n)
    np.matmul(b_c, a_c, out=out.reshape(n, cols, m))
    chat = out.reshape((m, cols) + a.shape[2:], order="F")
    return from_transform_domain(chat, mats)


def full_tsvdm_reconstruct(arr, mats):
    """full_tsvdm + TSVDMResult.reconstruct, tsvdm.py:190-202,236-243."""
    ahat = to_transform_domain(arr, mats)
    u, s, v = svd_all_slices(ahat)
    m, p = arr.shape[0], arr.shape[1]
    n = prod(arr.shape[2:])
    chat = np.empty((m, p, n), order="F")
    for i in range(n):
        chat[:, :, i] = (u[:, :, i] * s[:, i]) @ v[:, :, i].T
    return from_transform_domain(chat.reshape(arr.shape, order="F"), mats)


def rel_error(ref, other) -> float:
    """tests/helpers.py:44-47."""
    ref = np.asarray(ref).reshape(-1, order="F")
    other = np.asarray(other).reshape(-1, order="F")
    return float(np.linalg.norm(ref - other) / np.linalg.norm(ref))


def relative_error_from_energies(discarded, total) -> float:
    """CompressedTensor.relative_error, tsvdm.py:176-182."""
    if total == 0.0:
        return 0.0
    return math.sqrt(discarded / total)
