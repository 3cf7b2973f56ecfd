"""GPU parity of each kernel family against the CPU oracle (oracle/).

Run on a B200: ``pytest -m gpu``.  Every call goes through the public API
into libstarm.so; the oracle is only the checker.
"""

import math

import numpy as np
import pytest

import oracle
import paper_2605_16058_b200 as sb
from helpers import projector_distance, random_array, random_orthonormal, rel_error, sigma_close

pytestmark = pytest.mark.gpu

SHAPES = [(5, 3, 4), (3, 5, 2, 3), (7, 7, 6), (1, 4, 3), (4, 1, 2), (33, 17, 5), (17, 33, 4),
          (70, 130, 3), (130, 70, 3), (64, 64, 2), (200, 40, 3), (40, 200, 3), (2, 2, 2, 2, 3),
          (300, 257, 2), (257, 300, 2), (361, 720, 1), (1024, 1024, 2), (900, 1100, 1),
          (2100, 40, 2), (40, 2100, 2), (8192, 64, 2), (5000, 130, 1),
          # around the reduce kernel's update-path switch: L <= 960 keeps the
          # panel + team stage in SMEM (register team updates, widths 1..8);
          # longer slices use the SMEM-ring updates
          (1030, 200, 2), (200, 1030, 1), (520, 480, 1)]


# ------------------------------------------------------------------ TTM (K1)

@pytest.mark.parametrize("dims", [(3, 4, 5), (2, 3, 4, 2), (2, 2, 3, 2, 2), (3, 1, 4, 2),
                                  (16, 16, 64), (33, 5, 130), (7, 9, 257)])
def test_ttm_matches_oracle(dims):
    rng = np.random.default_rng(sum(dims))
    a = random_array(dims, sum(dims))
    t = sb.DenseTensor(a)
    for mode in range(2, len(dims)):
        for out_rows in (dims[mode], max(1, dims[mode] - 1), dims[mode] + 2):
            mat = rng.standard_normal((out_rows, dims[mode]))
            got = sb.ttm(t, mode, mat)
            ref = oracle.ttm(a, mode, mat)
            assert got.dims == ref.shape
            assert rel_error(ref, got.array) <= 1e-13


def test_ttm_large_dct_round_trip():
    dims = (37, 41, 96)
    a = random_array(dims, 3)
    t = sb.DenseTensor(a)
    ts = sb.TransformSet.build(dims, "dct")
    ahat = sb.to_transform_domain(t, ts)
    ref = oracle.to_transform_domain(a, [oracle.dct_matrix(96)])
    assert rel_error(ref, ahat.array) <= 1e-13
    back = sb.from_transform_domain(ahat, ts)
    assert rel_error(a, back.array) <= 1e-12
    assert abs(ahat.frobenius_norm() - t.frobenius_norm()) <= 1e-12 * t.frobenius_norm()


@pytest.mark.parametrize("dims,mode", [((37, 41, 2), 2), ((5, 3, 4), 2), ((3, 7, 8, 3), 2),
                                       ((2, 5, 3, 64), 3), ((9, 11, 1024), 2),
                                       ((3, 2, 2048), 2), ((2, 3, 4096), 2), ((1, 1, 16), 2),
                                       # n = 1024 register-FFT kernel: full tiles with 16-byte
                                       # access, an even-rows partial tile, batch > 1
                                       ((8, 12, 1024), 2), ((10, 13, 1024), 2),
                                       ((3, 4, 1024, 2), 2), ((1, 1, 1024), 2)])
def test_fast_dct_matches_dense_product(dims, mode):
    # the DCT kind applies the REFERENCE's operator: the dense DMMA product
    # with tr.matrix for n < 256, the FFT DCT plus the tcgen05 residual
    # (Delta = M - M_exact) from n = 256.  Either way the result is the
    # reference's dense product with its rounded dct_matrix to the rounding
    # of that product (~7e-16 Frobenius, numpy's own DGEMM error).
    a = random_array(dims, 17 + sum(dims))
    t = sb.DenseTensor(a)
    n = dims[mode]
    tr = sb.dct_matrix(n)
    got = sb.ttm(t, mode, tr)
    ref = oracle.ttm(a, mode, oracle.dct_matrix(n))
    assert rel_error(ref, got.array) <= 2e-15
    back = sb.ttm_inverse(got, mode, tr)
    ref_back = oracle.ttm(ref, mode, oracle.dct_matrix(n).T)
    assert rel_error(ref_back, back.array) <= 3e-15
    # the rounded M is not exactly orthonormal: the round trip's error is the
    # reference's own (~1e-13 at n = 1024), not the kernels'
    assert rel_error(a, back.array) <= 1.5 * rel_error(a, ref_back) + 1e-15


@pytest.mark.parametrize("n", [2, 4, 8, 16, 32, 64, 128, 256, 512, 1024, 2048, 4096])
def test_fft_dct_kernel_matches_exact_dct(n):
    # the raw FFT kernel (starm_dct_f64, C ABI) is the EXACT orthonormal
    # DCT-II / DCT-III: against scipy's FFT DCT to ~u log2 n
    import scipy.fft
    import torch
    from paper_2605_16058_b200 import _native as nat
    rows = 37 if n <= 1024 else 5
    a = random_array((rows, n), n)
    x = torch.from_numpy(a.reshape(-1, order="F").copy()).cuda()
    y = torch.empty_like(x)
    z = torch.empty_like(x)
    nat.call("starm_dct_f64", x.data_ptr(), y.data_ptr(), rows, n, 1, 0, nat.stream_ptr())
    nat.call("starm_dct_f64", y.data_ptr(), z.data_ptr(), rows, n, 1, 1, nat.stream_ptr())
    got = y.cpu().numpy().reshape((rows, n), order="F")
    exact = scipy.fft.dct(a, type=2, norm="ortho", axis=1)
    lg = max(1.0, math.log2(n))
    assert rel_error(exact, got) <= 2e-16 * lg + 1e-16
    assert rel_error(a, z.cpu().numpy().reshape((rows, n), order="F")) <= 4e-16 * lg + 1e-16


def test_dct_residual_kernel_direct():
    # starm_ttm_residual_bf16 alone: dst += 2^-e Delta_s @ src on the tensor
    # cores, against the float64 product (bf16 operands: ~3 digits of a
    # tiny term), partial fibre tiles and batch > 1
    import torch
    from paper_2605_16058_b200 import _native as nat
    rng = np.random.default_rng(5)
    for rows, n, batch in [(300, 256, 1), (129, 512, 2), (1000, 1024, 1), (7, 2048, 3)]:
        a = rng.standard_normal(rows * n * batch)
        delta = rng.standard_normal((n, n)) * 1e-14
        e = 46
        d_bf = torch.from_numpy(np.ldexp(delta, e)).to(torch.float32).to(torch.bfloat16).cuda()
        x = torch.from_numpy(a).cuda()
        base = rng.standard_normal(rows * n * batch)
        y = torch.from_numpy(base).cuda()
        lib = nat.load()
        nbytes = lib.starm_ttm_residual_workspace_bytes(rows, n, batch)
        ws = torch.empty(nbytes + 128, dtype=torch.uint8, device="cuda")
        p = ws.data_ptr() + (-ws.data_ptr()) % 128
        nat.call("starm_ttm_residual_bf16", x.data_ptr(), d_bf.data_ptr(), e, y.data_ptr(), rows, n,
                 batch, p, nbytes, nat.stream_ptr())
        got = y.cpu().numpy() - base
        ref = np.concatenate([(delta @ a[b * rows * n:(b + 1) * rows * n].reshape(n, rows)).ravel()
                              for b in range(batch)])
        assert np.linalg.norm(got - ref) <= 1e-2 * np.linalg.norm(ref), (rows, n, batch)


def test_fast_dct_rejects_non_power_of_two():
    from paper_2605_16058_b200 import _native as nat
    import torch
    x = torch.zeros(3 * 12, dtype=torch.float64, device="cuda")
    y = torch.empty_like(x)
    with pytest.raises(ValueError, match="power-of-two"):
        nat.call("starm_dct_f64", x.data_ptr(), y.data_ptr(), 3, 12, 1, 0, nat.stream_ptr())


# ------------------------------------------------------------- slice SVD (K3-K6)

@pytest.mark.parametrize("dims", SHAPES)
def test_svd_values_match_lapack(dims):
    a = random_array(dims, 7 + sum(dims))
    s = sb.svd_values_only(sb.DenseTensor(a))
    ref = oracle.svd_values_only(a)
    assert s.shape == ref.shape
    for i in range(ref.shape[1]):
        ok, excess = sigma_close(s[:, i], ref[:, i])
        assert ok, (dims, i, excess)


@pytest.mark.parametrize("dims", SHAPES)
def test_svd_full_factors(dims):
    a = random_array(dims, 11 + sum(dims))
    t = sb.DenseTensor(a)
    out = sb.svd_all_slices(t)
    m, p = dims[0], dims[1]
    r = min(m, p)
    n = t.num_slices
    assert out.u.dims == (m, r, n) and out.v.dims == (p, r, n) and out.s.shape == (r, n)
    values = sb.svd_values_only(t)
    assert np.array_equal(values, out.s)  # same rotation sequence -> bitwise
    for i in range(n):
        u = out.u.frontal_slice(i)
        v = out.v.frontal_slice(i)
        assert np.linalg.norm(u.T @ u - np.eye(r)) <= 1e-10 * math.sqrt(r)
        assert np.linalg.norm(v.T @ v - np.eye(r)) <= 1e-10 * math.sqrt(r)
        sl = t.frontal_slice(i)
        assert np.linalg.norm(out.reconstruct_slice(i) - sl) <= 1e-12 * np.linalg.norm(sl)
        assert (np.diff(out.s[:, i]) <= 0).all()


@pytest.mark.parametrize("dims", [(33, 17, 5), (17, 33, 4), (130, 70, 3), (64, 64, 2),
                                  (300, 257, 2), (361, 720, 1), (1500, 40, 2)])
def test_svd_subspaces_match_lapack(dims):
    # north_star: U / V compared by subspace (signs are arbitrary).  For every
    # k where the sigma gap is real, the projector distance between the
    # leading-k singular subspaces of the GPU and LAPACK stays within the
    # Wedin bound ~ c u sigma_max / gap.
    a = random_array(dims, 31 + sum(dims))
    out = sb.svd_all_slices(sb.DenseTensor(a))
    u_ref, s_ref, v_ref = oracle.svd_all_slices(a)
    r = min(dims[0], dims[1])
    ks = sorted(set([1, 2, 3, r // 4, r // 2, (3 * r) // 4, r - 1]))
    eps = np.finfo(float).eps
    for i in range(u_ref.shape[2]):
        s = s_ref[:, i]
        for k in ks:
            if k <= 0 or k >= r:
                continue
            gap = s[k - 1] - s[k]
            if gap <= 1e-8 * s[0]:
                continue
            bound = 1e-12 + 1024 * eps * s[0] / gap
            du = projector_distance(out.u.frontal_slice(i)[:, :k], u_ref[:, :k, i])
            dv = projector_distance(out.v.frontal_slice(i)[:, :k], v_ref[:, :k, i])
            assert du <= bound and dv <= bound, (i, k, du, dv, bound)


def test_zero_and_rank_deficient_slices():
    arr = np.zeros((4, 3, 2), order="F")
    arr[:, :, 1] = np.arange(12.0).reshape(4, 3)
    out = sb.svd_all_slices(sb.DenseTensor(arr, copy=False))
    assert np.array_equal(out.s[:, 0], np.zeros(3))
    assert np.array_equal(out.u.frontal_slice(0), np.eye(4, 3))
    assert np.array_equal(out.v.frontal_slice(0), np.eye(3, 3))
    u = out.u.frontal_slice(1)
    assert np.linalg.norm(u.T @ u - np.eye(3)) <= 1e-10 * math.sqrt(3)
    ref = oracle.svd_values_only(arr)
    ok, _ = sigma_close(out.s[:, 1], ref[:, 1])
    assert ok


def test_non_finite_slice_named():
    arr = np.zeros((3, 3, 5), order="F")
    arr[1, 1, 3] = np.nan
    arr[0, 0, 4] = np.inf
    t = sb.DenseTensor(arr, copy=False)
    with pytest.raises(ValueError, match="slice 3"):
        sb.svd_all_slices(t)
    with pytest.raises(ValueError, match="slice 3"):
        sb.svd_values_only(t)


def test_truncated_match_leading_triplets_bitwise():
    for dims in [(6, 5, 8), (5, 9, 8), (40, 70, 8)]:
        a = random_array(dims, 10)
        t = sb.DenseTensor(a)
        full = sb.svd_all_slices(t)
        r = min(dims[0], dims[1])
        ranks = np.array([0, 1, 2, 3, 4, r, 2, 1])
        f = sb.svd_truncated_slices(t, ranks)
        assert f.total_rank == int(ranks.sum())
        for i, k in enumerate(ranks):
            assert np.array_equal(f.u_block(i), full.u.frontal_slice(i)[:, :k])
            g = full.s[:k, i, None] * full.v.frontal_slice(i)[:, :k].T
            assert np.array_equal(f.g_block(i), g)


@pytest.mark.parametrize("dims,ranks", [((150, 170, 4), (0, 75, 150, 97)),
                                         ((420, 440, 3), (420, 33, 200))])
def test_truncated_bitwise_across_orth_blocks(dims, ranks):
    # r = 150: several 16-vector orthonormalisation blocks, earlier vectors
    # projected in more than one 64-column chunk, partial last blocks;
    # r = 420: also the DMMA LQ back-transformation (n > 400, 32-vector blocks)
    a = random_array(dims, 23)
    t = sb.DenseTensor(a)
    full = sb.svd_all_slices(t)
    r = min(dims[0], dims[1])
    ranks = np.array(ranks)
    f = sb.svd_truncated_slices(t, ranks)
    for i, k in enumerate(ranks):
        u = full.u.frontal_slice(i)
        v = full.v.frontal_slice(i)
        assert np.linalg.norm(u.T @ u - np.eye(r)) <= 1e-10 * math.sqrt(r)
        assert np.linalg.norm(v.T @ v - np.eye(r)) <= 1e-10 * math.sqrt(r)
        sl = t.frontal_slice(i)
        assert np.linalg.norm(full.reconstruct_slice(i) - sl) <= 1e-12 * np.linalg.norm(sl)
        assert np.array_equal(f.u_block(i), u[:, :k])
        g = full.s[:k, i, None] * full.v.frontal_slice(i)[:, :k].T
        assert np.array_equal(f.g_block(i), g)


def _degenerate_slices():
    """Slices whose singular values repeat exactly: blockdiag(B, B) (the two
    copies decouple in the bidiagonal), U diag(pairs) V^T, and rank-deficient
    traveling-Fourier-mode slices as in config c3 (cos/sin pairs)."""
    rng = np.random.default_rng(21)
    out = []
    for m, p in [(80, 60), (60, 80), (128, 128)]:
        b = rng.standard_normal((m // 2, p // 2))
        a = np.zeros((m, p))
        a[: m // 2, : p // 2] = b
        a[m // 2:, p // 2:] = b
        out.append(a)
        r = min(m, p)
        sig = np.repeat(np.linspace(3.0, 0.5, (r + 1) // 2), 2)[:r]
        u = np.linalg.qr(rng.standard_normal((m, r)))[0]
        v = np.linalg.qr(rng.standard_normal((p, r)))[0]
        out.append((u * sig) @ v.T)
    from paper_2605_16058_b200.configs import config3
    x, mm = config3(nx=128, ny=128, nt=16, modes=24, kmax=8)
    xh = oracle.ttm(x, 2, mm)
    out.extend(xh[:, :, i] for i in range(4))
    return out


@pytest.mark.parametrize("case", range(10))
def test_degenerate_spectrum_vectors(case):
    a = _degenerate_slices()[case]
    m, p = a.shape
    r = min(m, p)
    t = sb.DenseTensor(np.asfortranarray(a[:, :, None]))
    full = sb.svd_all_slices(t)
    u, v, s = full.u.frontal_slice(0), full.v.frontal_slice(0), full.s[:, 0]
    assert np.linalg.norm(u.T @ u - np.eye(r)) <= 1e-10 * math.sqrt(r)
    assert np.linalg.norm(v.T @ v - np.eye(r)) <= 1e-10 * math.sqrt(r)
    assert np.linalg.norm(full.reconstruct_slice(0) - a) <= 1e-12 * np.linalg.norm(a)
    ref = np.linalg.svd(a, compute_uv=False)
    for k in (1, 2, 3, 5, 8, 13, r // 2 + 1):
        f = sb.svd_truncated_slices(t, np.array([k]))
        err2 = np.sum((a - f.u_block(0) @ f.g_block(0)) ** 2)
        tail = np.sum(ref[k:] ** 2)
        assert abs(err2 - tail) <= 1e-9 * np.sum(ref ** 2), (k, err2, tail)


def test_graded_spectrum_values():
    # c5-like slice spectrum 0.8^j with Haar factors: analytic golden.
    rng = np.random.default_rng(5)
    m, p, n = 512, 64, 6
    arr = np.empty((m, p, n), order="F")
    sig = 0.8 ** np.arange(p)
    for i in range(n):
        u = np.linalg.qr(rng.standard_normal((m, p)))[0]
        v = np.linalg.qr(rng.standard_normal((p, p)))[0]
        arr[:, :, i] = (u * sig) @ v.T
    s = sb.svd_values_only(sb.DenseTensor(arr))
    ref = oracle.svd_values_only(arr)
    for i in range(n):
        ok, excess = sigma_close(s[:, i], ref[:, i])
        assert ok, excess
        assert np.max(np.abs(s[:, i] - sig) / sig) <= 1e-9


# ------------------------------------------------------------- threshold (K7)

def _threshold_equal(s, eps):
    got = sb.compute_threshold(s, eps)
    ref = oracle.compute_threshold(s, eps)
    assert np.array_equal(got.v, ref["v"])
    assert np.array_equal(got.w, ref["w"])
    assert got.j == ref["j"]
    assert got.tau == ref["tau"]
    assert np.array_equal(got.ranks, ref["ranks"])
    assert got.discarded_energy == ref["discarded_energy"]
    assert got.total_energy == ref["total_energy"]


def test_threshold_fixtures_bitwise():
    _threshold_equal(np.array([[3.0], [2.0], [1.0]]), 0.32)
    _threshold_equal(np.array([[2.0, 1.0], [1.0, 1.0]]), math.sqrt(2.5 / 7.0))
    _threshold_equal(np.array([[2.0], [1.0], [1.0]]), math.sqrt(2.5 / 6.0))
    _threshold_equal(np.array([[3.0], [1.0]]), 0.01)
    _threshold_equal(np.array([[3.0, 0.0], [1.0, 0.0]]), 0.01)
    th = sb.compute_threshold(np.zeros((3, 4)), 0.3)
    assert th.total_energy == 0.0 and th.tau == 0.0 and not th.ranks.any()


def test_threshold_random_bitwise():
    rng = np.random.default_rng(0)
    for trial in range(30):
        r, n = int(rng.integers(1, 40)), int(rng.integers(1, 300))
        s = -np.sort(-np.abs(rng.standard_normal((r, n))) * 10 ** rng.uniform(-3, 3, (1, n)), axis=0)
        for eps in (0.05, 0.2, 0.5, 0.9, 1e-3):
            _threshold_equal(np.asfortranarray(s), eps)


def test_threshold_ties_large():
    # many exact duplicates at the cutoff, > 128 dropped values (pairwise tree)
    rng = np.random.default_rng(3)
    vals = rng.choice(np.array([0.5, 1.0, 1.5, 2.0, 3.0]), size=(64, 500))
    s = -np.sort(-vals, axis=0)
    for eps in (0.1, 0.3, 0.5, 0.7):
        _threshold_equal(np.asfortranarray(s), eps)


# --------------------------------------------------------- end-to-end paths

def _kinds(dims, seed):
    return [sb.validate_transform(random_orthonormal(n, seed + k)) for k, n in enumerate(dims[2:])]


@pytest.mark.parametrize("dims", [(6, 5, 4, 2), (9, 13, 7), (20, 12, 16)])
def test_fixed_rank_matches_oracle(dims):
    a = random_array(dims, 4)
    t = sb.DenseTensor(a)
    for kinds in ("dct", "identity", "custom"):
        entries = _kinds(dims, 3) if kinds == "custom" else kinds
        ts = sb.TransformSet.build(dims, entries)
        mats = [tr.matrix for tr in ts]
        for rank in (1, 2, min(dims[0], dims[1])):
            c = sb.tsvdm_fixed_rank(t, ts, rank)
            ref = oracle.tsvdm_fixed_rank(a, mats, rank)
            assert np.array_equal(c.ranks, ref["ranks"])
            tot = ref["total_energy"]
            assert abs(c.total_energy - tot) <= 1e-12 * tot
            assert abs(c.discarded_energy - ref["discarded_energy"]) <= 1e-10 * tot
            rec = sb.reconstruct(c)
            rec_ref = oracle.reconstruct_packed(dims, mats, ref["ranks"], ref["u_data"], ref["g_data"])
            assert rel_error(rec_ref, rec.array) <= 1e-8
            err_sq = float(np.linalg.norm(rec.data - t.data) ** 2)
            assert abs(err_sq - ref["discarded_energy"]) <= 1e-10 * tot


@pytest.mark.parametrize("dims", [(5, 6, 4, 3), (12, 9, 10), (30, 50, 24)])
def test_tolerance_matches_oracle(dims):
    a = random_array(dims, 9)
    t = sb.DenseTensor(a)
    ts = sb.TransformSet.build(dims, "dct")
    mats = [tr.matrix for tr in ts]
    for eps in (0.4, 0.15, 0.05):
        ref = oracle.tsvdm_tolerance(a, mats, eps)
        recs = {}
        for strategy in (sb.TRUNCATE, sb.COMPUTE_EFFICIENT, sb.MEMORY_EFFICIENT):
            c = sb.tsvdm_tolerance(t, ts, eps, strategy=strategy)
            assert np.array_equal(c.ranks, ref["ranks"]), strategy
            recs[strategy] = sb.reconstruct(c)
            err = rel_error(a, recs[strategy].array)
            assert err < eps
            assert abs(c.relative_error() - err) <= 1e-8
        for strategy in recs:
            assert rel_error(recs[sb.TRUNCATE].array, recs[strategy].array) <= 1e-10


def test_dway_mixed_transforms_tolerance():
    # a 5-way tensor (the paper's datasets are 5-6-way) with
    # one transform kind per mode -- DCT (FFT path, n = 64), a custom Haar
    # matrix (DMMA GEMM path, middle mode: batch > 1) and the identity --
    # against the oracle: ranks bit-exact, energies, realised error.
    dims = (48, 40, 64, 6, 3)
    rng = np.random.default_rng(41)
    base = rng.standard_normal((48, 40, 4)) @ rng.standard_normal((4, 64 * 6 * 3))
    a = np.asfortranarray(base.reshape(dims, order="F") + 1e-2 * rng.standard_normal(dims))
    q, r = np.linalg.qr(rng.standard_normal((6, 6)))
    haar = sb.Transform(np.asfortranarray(q * np.sign(np.diag(r))), sb.CUSTOM)
    ts = sb.TransformSet.build(dims, [sb.DCT, haar, sb.IDENTITY])
    mats = [tr.matrix for tr in ts]
    t = sb.DenseTensor(a)
    for eps in (0.3, 0.02):
        ref = oracle.tsvdm_tolerance(a, mats, eps)
        c = sb.tsvdm_tolerance(t, ts, eps)
        assert np.array_equal(c.ranks, ref["ranks"])
        assert abs(c.discarded_energy - ref["discarded_energy"]) <= 1e-10 * ref["total_energy"]
        rec = sb.reconstruct(c)
        err = rel_error(a, rec.array)
        assert err < eps and abs(c.relative_error() - err) <= 1e-8


def test_tolerance_zero_tensor():
    t = sb.DenseTensor.zeros((4, 4, 3))
    ts = sb.TransformSet.build(t.dims, "identity")
    c = sb.tsvdm_tolerance(t, ts, 0.3)
    assert (c.ranks == 0).all()
    assert c.relative_error() == 0.0
    assert np.array_equal(sb.reconstruct(c).data, np.zeros(48))


def test_starm_product_matches_oracle():
    a = random_array((4, 3, 5, 2), 1)
    b = random_array((3, 6, 5, 2), 2)
    for kinds in ("identity", "dct"):
        ts = sb.TransformSet.build((4, 6, 5, 2), kinds)
        got = sb.starm_product(sb.DenseTensor(a), sb.DenseTensor(b), ts)
        ref = oracle.starm_product(a, b, [tr.matrix for tr in ts])
        assert rel_error(ref, got.array) <= 1e-12


def test_full_tsvdm_lossless():
    for dims in [(4, 5, 3), (3, 3, 2, 4), (5, 2, 3, 2, 2), (40, 30, 6)]:
        a = random_array(dims, 2)
        t = sb.DenseTensor(a)
        ts = sb.TransformSet.build(dims, "dct")
        res = sb.full_tsvdm(t, ts)
        assert rel_error(a, res.reconstruct().array) <= 1e-11


def test_tolerance_stream_equals_per_tensor_calls():
    dims = (30, 44, 16)
    ts = sb.TransformSet.build(dims, "dct")
    hosts = [sb.DenseTensor(random_array(dims, 40 + k)) for k in range(3)]
    got = list(sb.tsvdm_tolerance_stream(hosts, ts, 0.2))
    assert len(got) == 3
    for h, c in zip(hosts, got):
        ref = sb.tsvdm_tolerance(h, ts, 0.2)
        assert np.array_equal(c.ranks, ref.ranks)
        assert np.array_equal(c.factors.u_data, ref.factors.u_data)
        assert np.array_equal(c.factors.g_data, ref.factors.g_data)
        assert c.discarded_energy == ref.discarded_energy and c.total_energy == ref.total_energy
    assert list(sb.tsvdm_tolerance_stream([], ts, 0.2)) == []


@pytest.mark.parametrize("strategy", ["memory-efficient", "compute-efficient"])
def test_tolerance_on_tall_skinny_slices(strategy):
    # slices taller than the shared-memory panel (L > 1344): row-block TSQR
    # into stacked R factors, then the bidiagonal path (c5's 8192 x 64
    # slices take this route); both tolerance strategies
    dims = (1500, 24, 6)
    a = random_array(dims, 77)
    ts = sb.TransformSet.build(dims, "dct")
    got = sb.tsvdm_tolerance(sb.DenseTensor(a), ts, 0.05, strategy=strategy)
    ref = oracle.tsvdm_tolerance(a, [oracle.dct_matrix(6)], 0.05)
    assert np.array_equal(got.ranks, ref["ranks"])
    assert abs(got.discarded_energy - ref["discarded_energy"]) <= 1e-12 * ref["total_energy"]
    rec = sb.reconstruct(got)
    err = np.linalg.norm(rec.array - a) / np.linalg.norm(a)
    assert abs(err - got.relative_error()) <= 1e-8
