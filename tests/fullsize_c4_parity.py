"""Full-size c4 parity (not collected by pytest: minutes of CPU LAPACK).
GPU values / threshold from scripts/c4_dump.py vs the oracle restatement of
SURVEY 8c (float32 frames upcast to float64, raw non-orthonormal M, LAPACK
dgesvd values, compute_threshold at eps = 1e-3): sigma elementwise, the
threshold (J, tau) and the per-slice ranks (bit-exact).
usage: python tests/fullsize_c4_parity.py [gpurun_out/c4_gpu.npz] [procs]"""
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
    ahat = np.load("/tmp/c4_ahat.npy", mmap_mode="r")
    with threadpool_limits(limits=1, user_api="blas"):
        return lo, oracle.svd_values_only(np.asfortranarray(ahat[:, :, lo:hi]))


def main():
    import oracle
    from paper_2605_16058_b200.configs import config4
    path = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "gpurun_out", "c4_gpu.npz")
    procs = int(sys.argv[2]) if len(sys.argv) > 2 else os.cpu_count()
    g = np.load(path)
    t0 = time.time()
    a32, mm, _ = config4()
    a = np.asfortranarray(a32, dtype=np.float64)
    del a32
    ahat = oracle.ttm(a, 2, mm)
    del a
    np.save("/tmp/c4_ahat.npy", np.asfortranarray(ahat))
    n = ahat.shape[2]
    del ahat
    chunks = [(i, min(n, i + 16)) for i in range(0, n, 16)]
    s = np.zeros((512, n))
    with ProcessPoolExecutor(procs) as ex:
        for lo, part in ex.map(_values, chunks):
            s[:, lo:lo + part.shape[1]] = part
    th = oracle.compute_threshold(s, 1e-3)
    sg = g["s"]
    tol = 1e-10 * s + 64 * np.finfo(float).eps * s.max(axis=0, keepdims=True)
    bad = int((np.abs(sg - s) > tol).sum())
    ranks_ok = np.array_equal(th["ranks"], g["ranks"])
    q = s * s
    lines = [
        f"c4 full size (512x512x2048 f32 -> f64, M = I + 0.1 N/sqrt(n), eps 1e-3), oracle = ttm with the raw M + LAPACK dgesvd, {time.time() - t0:.0f} s on {procs} processes",
        f"sigma: elementwise violations of 1e-10 rel + 64u sigma_max floor: {bad} of {s.size}; max |ds| / sigma_max = {np.max(np.abs(sg - s) / s.max(axis=0, keepdims=True)):.3e}",
        f"threshold: J oracle {th['j']} gpu {int(g['j'])}, tau equal: {th['tau'] == float(g['tau'])}",
        f"ranks: sum oracle {int(th['ranks'].sum())}, sum gpu {int(g['ranks'].sum())}, bit-exact: {ranks_ok}",
        f"energies: total rel diff {abs(float(g['total']) - th['total_energy']) / th['total_energy']:.3e}, discarded rel diff {abs(float(g['discarded']) - th['discarded_energy']) / th['discarded_energy']:.3e}",
        f"threshold margin (sigma^2 other than tau itself): {np.min(np.abs(q[q != th['tau']] - th['tau'])) / th['tau']:.3e}",
    ]
    print("\n".join(lines))
    return 0 if ranks_ok and bad == 0 else 1


if __name__ == "__main__":
    sys.exit(main())
