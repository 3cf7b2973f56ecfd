"""Seeded synthetic stand-ins for the BASELINE.json configurations.

The paper's real datasets (NCEP reanalysis, CFD snapshots, X-ray frames,
PAPER.md:536,589,634) are not available; these generators reproduce the
shapes and value distributions BASELINE.json names.  Every draw happens in
a fixed, documented order from ``np.random.default_rng(seed)`` so the CPU
oracle and the GPU path see identical bytes.  All tensors are returned as
Fortran-ordered float64 (float32 for config 4) numpy arrays of shape
``(m, p, n)``.

Choices that BASELINE.json leaves open are fixed here:

* c1: factors a (m x R), b (p x R), c (n x R) ~ N(0,1) drawn in that order,
  then the noise as one flat column-major vector of length m*p*n.
* c2: 40 modes; per mode the draws are (degree l in [1,20], order
  mm in [0,l], cos/sin flag, c ~ N(0, l^-2), alpha, beta ~ N(0,1),
  phi, psi ~ U[0,2pi)) vectorised over modes in that order; Y is the real
  associated-Legendre harmonic P_l^mm(sin(lat)) * cos/sin(mm*lon)
  normalised to unit RMS over the grid; noise 1e-2*N(0,1) flat column-major.
* c3: 64 modes; integer wavevectors (kx, ky) with 1 <= |k| <= 32
  (rejection sampled), amplitude |k|^(-5/3), phase U[0,2pi), temporal
  frequency U[-0.05,0.05] cycles/step; M is Haar (QR of N(0,1) with the
  sign fix of tests/helpers.py:38-41), drawn after the modes.
* c4: Poisson(2) background, 200 Gaussian peaks (sigma 1.5 px, amplitude
  LogNormal(6,1), smooth per-frame profile 1 + 0.5 sin(2 pi t / T + phi),
  T ~ U[200, 2000]); M = I + 0.1 N(0,1)/sqrt(n); float32 storage.
* c5: per slice Haar U_i (m x p) and V_i (p x p), sigma_j = 0.8^j, M Haar;
  A = Ahat x_3 M^T.
"""

from __future__ import annotations

import math

import numpy as np

__all__ = [
    "haar_orthogonal", "dct_matrix_np", "config1", "config2", "config3",
    "config4", "config5_transform_domain", "CONFIGS",
]


def dct_matrix_np(n: int) -> np.ndarray:
    """Orthonormal DCT-II (same formula as transforms.dct_matrix)."""
    j = np.arange(n)[:, None]
    k = np.arange(n)[None, :]
    mat = np.cos(np.pi * (2 * k + 1) * j / (2.0 * n))
    mat[0, :] *= np.sqrt(1.0 / n)
    if n > 1:
        mat[1:, :] *= np.sqrt(2.0 / n)
    return np.asfortranarray(mat)


def haar_orthogonal(n: int, rng: np.random.Generator, cols: int | None = None) -> np.ndarray:
    """QR of an N(0,1) matrix with the diagonal-sign fix (tests/helpers.py:38-41)."""
    cols = n if cols is None else cols
    q, r = np.linalg.qr(rng.standard_normal((n, cols)))
    return np.asfortranarray(q * np.sign(np.diag(r)))


def config1(m=256, p=256, n=64, rank=10, noise=1e-3, seed=0):
    """c1: sum of ``rank`` rank-1 outer products + noise.  M = DCT-II(n),
    truncate every slice to rank 10."""
    rng = np.random.default_rng(seed)
    a = rng.standard_normal((m, rank))
    b = rng.standard_normal((p, rank))
    c = rng.standard_normal((n, rank))
    x = np.einsum("ir,jr,kr->ijk", a, b, c, optimize=True)
    x = np.asfortranarray(x)
    x += noise * rng.standard_normal(m * p * n).reshape((m, p, n), order="F")
    return x


def _assoc_legendre(l, mm, x):
    from scipy.special import lpmv
    return lpmv(mm, l, x)


def config2(nlat=361, nlon=720, nt=1024, modes=40, max_degree=20, noise=1e-2, seed=0):
    """c2: climate-reanalysis-like field, lat x lon x time, DCT over time,
    tolerance 1e-2."""
    rng = np.random.default_rng(seed)
    deg = rng.integers(1, max_degree + 1, size=modes)
    order = np.array([rng.integers(0, l + 1) for l in deg])
    use_sin = rng.integers(0, 2, size=modes)
    coef = rng.standard_normal(modes) / deg
    alpha = rng.standard_normal(modes)
    beta = rng.standard_normal(modes)
    phi = rng.uniform(0.0, 2 * np.pi, size=modes)
    psi = rng.uniform(0.0, 2 * np.pi, size=modes)
    lat = np.deg2rad(np.linspace(-90.0, 90.0, nlat))
    lon = np.deg2rad(np.arange(nlon) * (360.0 / nlon))
    spatial = np.empty((nlat * nlon, modes), order="F")
    for k in range(modes):
        pl = _assoc_legendre(int(deg[k]), int(order[k]), np.sin(lat))
        az = np.sin(order[k] * lon) if (use_sin[k] and order[k] > 0) else np.cos(order[k] * lon)
        y = np.outer(pl, az)
        rms = math.sqrt(float(np.mean(y * y)))
        y = y / rms if rms > 0 else y
        spatial[:, k] = coef[k] * y.reshape(-1, order="F")
    t = np.arange(nt)
    temporal = (alpha[:, None] * np.sin(2 * np.pi * t[None, :] / 365.0 + phi[:, None])
                + beta[:, None] * np.sin(2 * np.pi * t[None, :] / 182.0 + psi[:, None]))
    x = spatial @ temporal  # (nlat*nlon, nt), column-major == F-order tensor
    x = np.asfortranarray(x)
    x += noise * rng.standard_normal(x.size).reshape(x.shape, order="F")
    return x.reshape((nlat, nlon, nt), order="F")


def config3(nx=1024, ny=1024, nt=512, modes=64, kmax=32, seed=0):
    """c3: CFD-like traveling Fourier modes; M = Haar(nt); rank 32.
    Returns (tensor, M)."""
    rng = np.random.default_rng(seed)
    ks = []
    while len(ks) < modes:
        kx, ky = rng.integers(-kmax, kmax + 1, size=2)
        mag = math.hypot(kx, ky)
        if 1 <= mag <= kmax:
            ks.append((int(kx), int(ky)))
    ks = np.array(ks, dtype=np.float64)
    amp = np.hypot(ks[:, 0], ks[:, 1]) ** (-5.0 / 3.0)
    phase = rng.uniform(0, 2 * np.pi, size=modes)
    freq = rng.uniform(-0.05, 0.05, size=modes)
    xs = np.arange(nx) * (2 * np.pi / nx)
    ys = np.arange(ny) * (2 * np.pi / ny)
    t = np.arange(nt)
    # cos(kx x + ky y + phi - 2 pi f t) = Re(S_q(x) * T_q(t))
    sx = np.exp(1j * np.outer(xs, ks[:, 0]))            # (nx, modes)
    sy = np.exp(1j * np.outer(ys, ks[:, 1]))            # (ny, modes)
    s = (sx[:, None, :] * sy[None, :, :]).reshape(nx * ny, modes, order="F")
    s = s * (amp * np.exp(1j * phase))[None, :]
    tt = np.exp(-2j * np.pi * np.outer(freq, t))        # (modes, nt)
    x = s.real @ tt.real - s.imag @ tt.imag
    m = haar_orthogonal(nt, rng)
    return np.asfortranarray(x).reshape((nx, ny, nt), order="F"), m


def config4(nx=512, ny=512, nt=2048, peaks=200, lam=2.0, seed=0):
    """c4: X-ray-like frames, float32.  Returns (tensor_f32, M, M_inv)."""
    rng = np.random.default_rng(seed)
    bg = rng.poisson(lam, size=nx * ny * nt).astype(np.float32)
    cx = rng.uniform(0, nx, size=peaks)
    cy = rng.uniform(0, ny, size=peaks)
    amp = rng.lognormal(6.0, 1.0, size=peaks)
    period = rng.uniform(200.0, 2000.0, size=peaks)
    ph = rng.uniform(0, 2 * np.pi, size=peaks)
    xs = np.arange(nx)[:, None]
    ys = np.arange(ny)[None, :]
    spatial = np.empty((nx * ny, peaks), order="F")
    for q in range(peaks):
        g = np.exp(-((xs - cx[q]) ** 2 + (ys - cy[q]) ** 2) / (2 * 1.5 ** 2))
        spatial[:, q] = amp[q] * g.reshape(-1, order="F")
    t = np.arange(nt)
    temporal = 1.0 + 0.5 * np.sin(2 * np.pi * t[None, :] / period[:, None] + ph[:, None])
    x = (spatial @ temporal).astype(np.float32)
    x += bg.reshape(x.shape, order="F")
    mmat = np.eye(nt) + 0.1 * rng.standard_normal((nt, nt)) / math.sqrt(nt)
    minv = np.linalg.inv(mmat)
    return (np.asfortranarray(x).reshape((nx, ny, nt), order="F"),
            np.asfortranarray(mmat), np.asfortranarray(minv))


def config5_transform_domain(m=8192, p=64, n=4096, decay=0.8, seed=0):
    """c5 in the M domain: Ahat_i = U_i diag(decay^j) V_i^T; returns
    (ahat, M).  The original-domain tensor is ttm(ahat, 2, M^T)."""
    rng = np.random.default_rng(seed)
    sig = decay ** np.arange(p)
    ahat = np.empty((m, p, n), order="F")
    for i in range(n):
        u = haar_orthogonal(m, rng, cols=p)
        v = haar_orthogonal(p, rng)
        ahat[:, :, i] = (u * sig) @ v.T
    mmat = haar_orthogonal(n, rng)
    return ahat, mmat


def config5_fibre_block(f0, f1, m=8192, p=64, n=4096, decay=0.8, seed=0):
    """Fibres [f0, f1) of config5_transform_domain's Ahat as an (f1 - f0, n)
    float64 array (row = fibre, column = slice), plus M -- the same draws in
    the same order, without the full m*p*n tensor (a rank of the sharded
    bench holds only its fibre block)."""
    rng = np.random.default_rng(seed)
    sig = decay ** np.arange(p)
    out = np.empty((f1 - f0, n), order="F")
    for i in range(n):
        u = haar_orthogonal(m, rng, cols=p)
        v = haar_orthogonal(p, rng)
        sl = (u * sig) @ v.T
        out[:, i] = sl.reshape(-1, order="F")[f0:f1]
    mmat = haar_orthogonal(n, rng)
    return out, mmat


CONFIGS = {
    "c1": dict(kind="fixed-rank", rank=10, dims=(256, 256, 64), transform="dct"),
    "c2": dict(kind="tolerance", epsilon=1e-2, dims=(361, 720, 1024), transform="dct"),
    "c3": dict(kind="fixed-rank", rank=32, dims=(1024, 1024, 512), transform="haar"),
    "c4": dict(kind="tolerance", epsilon=1e-3, dims=(512, 512, 2048), transform="invertible"),
    "c5": dict(kind="fixed-rank+tolerance", rank=16, epsilon=1e-4, dims=(8192, 64, 4096),
               transform="haar"),
}
