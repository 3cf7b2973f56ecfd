"""Golden-case definitions shared by make_golden.py (reference side) and the
parity tests (oracle / CUDA side).  Inputs are regenerated from these seeds."""

import math
from math import prod

import numpy as np


def make_tensor(dims, seed):
    rng = np.random.default_rng(seed)
    return rng.standard_normal(prod(dims)).reshape(dims, order="F")


def random_orthonormal(n, seed):
    rng = np.random.default_rng(seed)
    q, r = np.linalg.qr(rng.standard_normal((n, n)))
    return q * np.sign(np.diag(r))


def make_transforms(mod, dims, kind, seed):
    """Transform spec for TransformSet.build of module ``mod`` (starm or ours)."""
    if kind == "custom":
        return [mod.validate_transform(random_orthonormal(n, seed + 7 + k))
                for k, n in enumerate(dims[2:])]
    return kind


def _decaying(r, n, seed):
    rng = np.random.default_rng(seed)
    s = np.abs(rng.standard_normal((r, n))) * (10.0 ** -rng.uniform(0, 4, (r, 1)))
    return -np.sort(-s, axis=0)


def _ties(seed):
    rng = np.random.default_rng(seed)
    vals = rng.choice(np.array([0.25, 0.5, 1.0, 2.0]), size=(48, 300))
    return -np.sort(-vals, axis=0)


THRESHOLD_CASES = {
    "fixture_a2": (np.array([[3.0], [2.0], [1.0]]), 0.32),
    "ties_retained": (np.array([[2.0, 1.0], [1.0, 1.0]]), math.sqrt(2.5 / 7.0)),
    "ties_dropped": (np.array([[2.0], [1.0], [1.0]]), math.sqrt(2.5 / 6.0)),
    "budget_below_min": (np.array([[3.0], [1.0]]), 0.01),
    "exact_zeros": (np.array([[3.0, 0.0], [1.0, 0.0]]), 0.01),
    "all_zero": (np.zeros((3, 4)), 0.3),
    "decaying_64x400": (_decaying(64, 400, 1), 1e-2),
    "decaying_361x100": (_decaying(361, 100, 2), 1e-3),
    "ties_48x300_a": (_ties(3), 0.3),
    "ties_48x300_b": (_ties(4), 0.6),
}

TTM_CASES = {
    "3way_m2": ((3, 4, 5), 1, 2, 5),
    "3way_m2_wide": ((6, 5, 9), 2, 2, 11),
    "4way_m2": ((2, 3, 4, 2), 3, 2, 3),
    "4way_m3": ((2, 3, 4, 2), 4, 3, 2),
    "5way_m3": ((2, 2, 3, 2, 2), 5, 3, 4),
    "deg_1": ((3, 1, 4, 2), 6, 2, 4),
}

SVD_CASES = {
    "tall": ((7, 5, 6), 3),
    "wide": ((5, 8, 4), 4),
    "square": ((6, 6, 3), 5),
    "4way": ((5, 3, 4, 2), 1),
    "mid": ((40, 24, 3), 6),
}

FIXED_RANK_CASES = {
    "dct_r1": ((6, 5, 4, 2), 0, "dct", 1),
    "id_r2": ((6, 5, 4, 2), 1, "identity", 2),
    "custom_r4": ((6, 5, 4, 2), 2, "custom", 4),
    "dct_wide_r3": ((5, 7, 3, 2), 3, "dct", 3),
    "dct_5way_r2": ((4, 4, 2, 2, 3), 4, "dct", 2),
}

TOLERANCE_CASES = {
    "dct_040": ((5, 6, 4, 3), 0, "dct", 0.4),
    "dct_015": ((5, 6, 4, 3), 1, "dct", 0.15),
    "id_015": ((5, 6, 4, 3), 2, "identity", 0.15),
    "custom_040": ((6, 5, 8), 3, "custom", 0.4),
    "dct_020_mid": ((30, 20, 16), 4, "dct", 0.2),
}

PRODUCT_CASES = {
    "identity": ((4, 3, 5, 2), (3, 6, 5, 2), 1, "identity"),
    "dct": ((4, 3, 5, 2), (3, 6, 5, 2), 2, "dct"),
    "dct_3way": ((3, 4, 6), (4, 5, 6), 3, "dct"),
}
