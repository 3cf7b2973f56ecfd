"""Generate the golden fixtures that pin oracle/ to the reference package.

Run IN THE BUILD CONTAINER ONLY (it imports the read-only reference at
/root/reference/pkg/src, which does not exist on the GPU box):

    python tests/golden/make_golden.py

Every case runs the reference package itself (`starm`) and stores inputs
seeds + outputs in tests/golden/golden.npz.  tests/test_oracle_golden.py
then checks the oracle restatement (and, on a GPU, tests/test_gpu_golden.py
checks the CUDA path) against these outputs.  Inputs are regenerated from
the committed seeds/generators, so only outputs are stored.
"""

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, "/root/reference/pkg/src")

import starm  # noqa: E402  (reference, read-only)

from tests.golden.cases import (THRESHOLD_CASES, TOLERANCE_CASES, FIXED_RANK_CASES, TTM_CASES,  # noqa: E402
                                SVD_CASES, PRODUCT_CASES, make_tensor, make_transforms)


def main():
    out = {}
    # --- compute_threshold (tsvdm.py:85-115): exact outputs
    for name, (s, eps) in THRESHOLD_CASES.items():
        th = starm.compute_threshold(s, eps)
        out[f"th/{name}/v"] = th.v
        out[f"th/{name}/w"] = th.w
        out[f"th/{name}/j"] = np.array(th.j)
        out[f"th/{name}/tau"] = np.array(th.tau)
        out[f"th/{name}/ranks"] = th.ranks
        out[f"th/{name}/disc"] = np.array(th.discarded_energy)
        out[f"th/{name}/total"] = np.array(th.total_energy)
    # --- ttm (ttm.py:87-135)
    for name, (dims, seed, mode, rows) in TTM_CASES.items():
        t = make_tensor(dims, seed)
        mat = np.random.default_rng(seed + 1).standard_normal((rows, dims[mode]))
        out[f"ttm/{name}"] = starm.ttm(starm.DenseTensor(t), mode, mat).array
    # --- slice SVD values + factors (slicesvd.py:115-177)
    for name, (dims, seed) in SVD_CASES.items():
        t = starm.DenseTensor(make_tensor(dims, seed))
        res = starm.svd_all_slices(t)
        out[f"svd/{name}/s"] = res.s
        out[f"svd/{name}/u"] = res.u.array
        out[f"svd/{name}/v"] = res.v.array
    # --- fixed rank (tsvdm.py:246-265)
    for name, (dims, seed, kind, rank) in FIXED_RANK_CASES.items():
        t = starm.DenseTensor(make_tensor(dims, seed))
        ts = starm.TransformSet.build(dims, make_transforms(starm, dims, kind, seed))
        c = starm.tsvdm_fixed_rank(t, ts, rank)
        out[f"fr/{name}/ranks"] = c.ranks
        out[f"fr/{name}/disc"] = np.array(c.discarded_energy)
        out[f"fr/{name}/total"] = np.array(c.total_energy)
        out[f"fr/{name}/recon"] = starm.reconstruct(c).array
        out[f"fr/{name}/u"] = c.factors.u_data
        out[f"fr/{name}/g"] = c.factors.g_data
    # --- tolerance (tsvdm.py:268-321) for all three strategies (identical)
    for name, (dims, seed, kind, eps) in TOLERANCE_CASES.items():
        t = starm.DenseTensor(make_tensor(dims, seed))
        ts = starm.TransformSet.build(dims, make_transforms(starm, dims, kind, seed))
        c = starm.tsvdm_tolerance(t, ts, eps)
        out[f"tol/{name}/ranks"] = c.ranks
        out[f"tol/{name}/disc"] = np.array(c.discarded_energy)
        out[f"tol/{name}/total"] = np.array(c.total_energy)
        out[f"tol/{name}/recon"] = starm.reconstruct(c).array
        out[f"tol/{name}/s"] = starm.svd_values_only(starm.to_transform_domain(t, ts))
    # --- *_M product (tsvdm.py:219-233)
    for name, (da, db, seed, kind) in PRODUCT_CASES.items():
        a = starm.DenseTensor(make_tensor(da, seed))
        b = starm.DenseTensor(make_tensor(db, seed + 1))
        ts = starm.TransformSet.build((da[0], db[1]) + tuple(da[2:]), kind)
        out[f"prod/{name}"] = starm.starm_product(a, b, ts).array
    np.savez_compressed(os.path.join(HERE, "golden.npz"), **out)
    print(f"wrote {len(out)} arrays to tests/golden/golden.npz")
    configs()


def configs():
    """Config-level goldens (BASELINE.json configs at full or reduced scale)."""
    from paper_2605_16058_b200 import configs as cf
    out = {}
    # c1 at full size: 256x256x64, DCT, rank 10 (BASELINE configs[0])
    a = cf.config1()
    t = starm.DenseTensor(a)
    ts = starm.TransformSet.build(a.shape, "dct")
    c = starm.tsvdm_fixed_rank(t, ts, 10)
    rec = starm.reconstruct(c)
    out["c1/ranks"] = c.ranks
    out["c1/disc"] = np.array(c.discarded_energy)
    out["c1/total"] = np.array(c.total_energy)
    out["c1/relerr"] = np.array(np.linalg.norm(rec.data - t.data) / np.linalg.norm(t.data))
    out["c1/s"] = starm.svd_values_only(starm.to_transform_domain(t, ts))
    out["c1/u0"] = c.factors.u_block(0).copy()
    out["c1/g0"] = c.factors.g_block(0).copy()
    # c2 reduced: 91 x 180 x 128, DCT, tolerance 1e-2
    a = cf.config2(nlat=91, nlon=180, nt=128)
    t = starm.DenseTensor(a)
    ts = starm.TransformSet.build(a.shape, "dct")
    vals = starm.svd_values_only(starm.to_transform_domain(t, ts))
    th = starm.compute_threshold(vals, 1e-2)
    c = starm.tsvdm_tolerance(t, ts, 1e-2)
    out["c2r/s"] = vals
    out["c2r/ranks"] = c.ranks
    out["c2r/j"] = np.array(th.j)
    out["c2r/tau"] = np.array(th.tau)
    out["c2r/disc"] = np.array(c.discarded_energy)
    out["c2r/total"] = np.array(c.total_energy)
    out["c2r/relerr"] = np.array(np.linalg.norm(starm.reconstruct(c).data - t.data)
                                 / np.linalg.norm(t.data))
    # c5 reduced: 512 x 64 x 128, sigma_j = 0.8^j, Haar M; rank 16 and tol 1e-4
    ahat, mmat = cf.config5_transform_domain(m=512, p=64, n=128)
    a = starm.ttm(starm.DenseTensor(ahat), 2, mmat.T).array
    t = starm.DenseTensor(a)
    ts = starm.TransformSet((starm.validate_transform(mmat),))
    c16 = starm.tsvdm_fixed_rank(t, ts, 16)
    ct = starm.tsvdm_tolerance(t, ts, 1e-4)
    vals = starm.svd_values_only(starm.to_transform_domain(t, ts))
    out["c5r/s"] = vals
    out["c5r/fr_disc"] = np.array(c16.discarded_energy)
    out["c5r/fr_total"] = np.array(c16.total_energy)
    out["c5r/tol_ranks"] = ct.ranks
    out["c5r/tol_disc"] = np.array(ct.discarded_energy)
    np.savez_compressed(os.path.join(HERE, "golden_configs.npz"), **out)
    print(f"wrote {len(out)} arrays to tests/golden/golden_configs.npz")


if __name__ == "__main__":
    main()


def datadriven():
    """Reference data_driven_transform (transforms.py:94-110) on seeded tensors,
    and a tolerance t-SVDM over it -> tests/golden/golden_datadriven.npz."""
    out = {}
    cases = {"3way": ((12, 9, 16), 2, 21), "wide_rest": ((3, 2, 12), 2, 22), "4way_m3": ((4, 5, 3, 10), 3, 23)}
    for name, (dims, mode, seed) in cases.items():
        rng = np.random.default_rng(seed)
        a = np.asfortranarray(rng.standard_normal(dims) * np.logspace(0, -1, dims[mode]).reshape(
            [dims[mode] if k == mode else 1 for k in range(len(dims))]))
        tr = starm.data_driven_transform(starm.DenseTensor(a), mode)
        out[f"{name}/m"] = tr.matrix
    rng = np.random.default_rng(30)
    a = np.asfortranarray(rng.standard_normal((10, 12, 24)) + np.einsum(
        "i,j,k->ijk", rng.standard_normal(10), rng.standard_normal(12), rng.standard_normal(24)) * 3)
    t = starm.DenseTensor(a)
    ts = starm.TransformSet.build(a.shape, "data-driven", tensor=t)
    c = starm.tsvdm_tolerance(t, ts, 0.2)
    out["tol/ranks"] = c.ranks
    out["tol/disc"] = np.array(c.discarded_energy)
    out["tol/total"] = np.array(c.total_energy)
    out["tol/s"] = starm.svd_values_only(starm.to_transform_domain(t, ts))
    np.savez_compressed(os.path.join(HERE, "golden_datadriven.npz"), **out)
    print(f"wrote {len(out)} arrays to tests/golden/golden_datadriven.npz")
