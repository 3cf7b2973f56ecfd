"""Seeded inputs shared by the tests (mirrors the reference's
tests/helpers.py:16-47 input recipes)."""

from math import prod

import numpy as np


def random_array(dims, seed):
    rng = np.random.default_rng(seed)
    return rng.standard_normal(prod(dims)).reshape(dims, order="F")


def random_orthonormal(n, seed):
    rng = np.random.default_rng(seed)
    q, r = np.linalg.qr(rng.standard_normal((n, n)))
    return q * np.sign(np.diag(r))


def rel_error(ref, other):
    ref = np.asarray(ref).reshape(-1, order="F")
    other = np.asarray(other).reshape(-1, order="F")
    return float(np.linalg.norm(ref - other) / np.linalg.norm(ref))


def sigma_close(got, ref, rtol=1e-10, floor=64.0):
    """|dsigma_i| <= rtol*sigma_i + floor*u*sigma_max (SURVEY 8d parity bar)."""
    got = np.asarray(got)
    ref = np.asarray(ref)
    smax = float(np.max(ref)) if ref.size else 0.0
    tol = rtol * ref + floor * np.finfo(float).eps * smax
    return bool(np.all(np.abs(got - ref) <= tol)), float(np.max(np.abs(got - ref) - tol)) if ref.size else 0.0


def projector_distance(u1, u2):
    """||U1 U1^T - U2 U2^T||_2 for orthonormal column blocks."""
    d = u1 @ u1.T - u2 @ u2.T
    return float(np.linalg.norm(d, 2)) if d.size else 0.0
