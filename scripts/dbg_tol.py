import sys
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import numpy as np
import paper_2605_16058_b200 as sb
import oracle
from helpers import random_array, rel_error
dims = (5, 6, 4, 3)
a = random_array(dims, 9)
t = sb.DenseTensor(a)
ts = sb.TransformSet.build(dims, "dct")
mats = [tr.matrix for tr in ts]
for eps in (0.4, 0.15):
    ref = oracle.tsvdm_tolerance(a, mats, eps)
    for strategy in (sb.TRUNCATE, sb.COMPUTE_EFFICIENT, sb.MEMORY_EFFICIENT):
        c = sb.tsvdm_tolerance(t, ts, eps, strategy=strategy)
        rec = sb.reconstruct(c)
        print(eps, strategy, c.ranks.tolist(), rel_error(a, rec.array), np.abs(c.factors.g_data - ref["g_data"]).max() if c.factors.g_data.size == ref["g_data"].size else "size")
        ro = oracle.reconstruct_packed(dims, mats, c.ranks, c.factors.u_data, c.factors.g_data)
        print("   oracle-recon of our factors:", rel_error(a, ro))
