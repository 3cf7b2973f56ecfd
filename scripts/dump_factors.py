"""Hash of the packed factors of fixed small problems (bitwise regression
check across kernel changes): prints sha256 of u_data / g_data."""
import hashlib, sys
import numpy as np, torch
sys.path.insert(0, ".")
import paper_2605_16058_b200 as sb
rng = np.random.default_rng(7)
for dims, eps in (((37, 52, 64), 0.2), ((64, 48, 256), 0.05), ((300, 257, 8), 0.3)):
    a = np.asfortranarray(rng.standard_normal(dims).cumsum(axis=2))
    ts = sb.TransformSet.build(dims, "dct")
    c = sb.tsvdm_tolerance(sb.DenseTensor(a), ts, eps)
    f = c.factors
    print(dims, int(c.ranks.sum()), hashlib.sha256(f.u_data.tobytes()).hexdigest()[:16], hashlib.sha256(f.g_data.tobytes()).hexdigest()[:16])
    r = sb.tsvdm_fixed_rank(sb.DenseTensor(a), ts, min(dims[0], dims[1]) // 2)
    print("   fixed", hashlib.sha256(r.factors.u_data.tobytes()).hexdigest()[:16], hashlib.sha256(r.factors.g_data.tobytes()).hexdigest()[:16])
