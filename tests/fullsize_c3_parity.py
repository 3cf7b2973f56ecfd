"""Full-size c3 parity (not collected by pytest: ~15 min of CPU LAPACK on 8
processes).  GPU values from scripts/c3_dump.py vs the oracle (dense Haar
transform + LAPACK dgesvd per slice): singular values elementwise within
1e-10 relative above a 64u sigma_max floor, and the fixed-rank energies.
usage: python tests/fullsize_c3_parity.py [gpurun_out/c3_gpu.npz] [procs]"""
import os
import sys
import time
from concurrent.futures import ProcessPoolExecutor

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def _values(args):
    lo, hi = args
    from threadpoolctl import threadpool_limits
    import oracle
    ahat = np.load("/tmp/c3_ahat.npy", mmap_mode="r")
    with threadpool_limits(limits=1, user_api="blas"):
        return lo, oracle.svd_values_only(np.asfortranarray(ahat[:, :, lo:hi]))


def main():
    import oracle
    from paper_2605_16058_b200.configs import config3
    path = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "gpurun_out", "c3_gpu.npz")
    procs = int(sys.argv[2]) if len(sys.argv) > 2 else os.cpu_count()
    g = np.load(path)
    t0 = time.time()
    a, mm = config3()
    ahat = oracle.to_transform_domain(a, [mm])
    del a
    np.save("/tmp/c3_ahat.npy", np.asfortranarray(ahat))
    n = ahat.shape[2]
    del ahat
    chunks = [(i, min(n, i + 4)) for i in range(0, n, 4)]
    s = np.zeros((1024, n))
    with ProcessPoolExecutor(procs) as ex:
        for lo, part in ex.map(_values, chunks):
            s[:, lo:lo + part.shape[1]] = part
    sg = g["s"]
    smax = s.max(axis=0, keepdims=True)
    tol = 1e-10 * s + 64 * np.finfo(float).eps * smax
    bad = int((np.abs(sg - s) > tol).sum())
    lead = np.max(np.abs(sg[:32] - s[:32]) / s[:32])
    total = float(np.sum(s * s))
    disc = float(np.sum(s[32:] * s[32:]))
    lines = [
        f"c3 full size (1024x1024x512, Haar M, rank 32), oracle = dense transform + LAPACK dgesvd, {time.time() - t0:.0f} s on {procs} processes",
        f"sigma: elementwise violations of 1e-10 rel + 64u sigma_max floor: {bad} of {s.size}; leading 32 max rel diff {lead:.3e}",
        f"energies: total rel diff {abs(float(g['total']) - total) / total:.3e}, discarded rel diff {abs(float(g['discarded']) - disc) / disc:.3e}",
    ]
    print("\n".join(lines))
    return 0 if bad == 0 else 1


if __name__ == "__main__":
    sys.exit(main())
