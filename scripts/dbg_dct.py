import sys
import numpy as np
import scipy.fft
sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import oracle
import paper_2605_16058_b200 as sb
from helpers import random_array, rel_error
for dims in [(9, 11, 1024), (3, 2, 2048), (2, 5, 64), (37, 41, 2)]:
    n = dims[2]
    a = random_array(dims, 17 + sum(dims))
    t = sb.DenseTensor(a)
    tr = sb.dct_matrix(n)
    got = sb.ttm(t, 2, tr).array
    ref = oracle.ttm(a, 2, oracle.dct_matrix(n))
    exact = scipy.fft.dct(a, type=2, norm="ortho", axis=2)
    back = sb.ttm_inverse(sb.DenseTensor(got), 2, tr).array
    eback = scipy.fft.idct(exact, type=2, norm="ortho", axis=2)
    print(dims, "fwd ours-scipy %.2e dense-scipy %.2e | inv ours-a %.2e scipy-a %.2e"
          % (rel_error(exact, got), rel_error(exact, ref), rel_error(a, back), rel_error(a, eback)))
