"""Codec fixtures written by the reference package itself (section 8(f) f1).

Run IN THE BUILD CONTAINER ONLY (imports /root/reference/pkg/src):

    python tests/golden/make_codec_golden.py

Writes tests/golden/codec_golden.json: the hex bytes the reference's
write_tensor / write_compressed (codec.py:142-189) produce for
  * ten_small: DenseTensor(arange(8), (2, 2, 2));
  * cmp_small: dims (2, 2, 2), tsvdm2 param 0.5, identity transform,
    ranks (1, 0), U block [1, 2], G block [3, 4];
  * cmp_mixed: tsvdm_tolerance(eps 0.35) of a seeded (5, 4, 3, 2) tensor
    with a data-driven mode-2 and a custom (seeded orthonormal) mode-3
    transform (stored matrices, variable ranks);
  * cmp_dct: tsvdm_fixed_rank(rank 2) of a seeded (6, 5, 8) tensor with DCT
    (regenerated transform), and the input tensor itself (ten_dct).
tests/test_codec.py reads these with paper_2605_16058_b200.codec and checks
read -> write reproduces every byte.
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

import starm  # noqa: E402  (reference, read-only)


def hexof(writer, obj):
    import io
    buf = io.BytesIO()
    writer(obj, buf)
    return buf.getvalue().hex()


def orthonormal(n, seed):
    q, r = np.linalg.qr(np.random.default_rng(seed).standard_normal((n, n)))
    return q * np.sign(np.diag(r))


def main():
    out = {}
    out["ten_small"] = hexof(starm.write_tensor, starm.DenseTensor(np.arange(8.0), (2, 2, 2), copy=False))
    f = starm.VariableRankFactors(2, 2, np.array([1, 0]), np.array([1.0, 2.0]), np.array([3.0, 4.0]))
    c = starm.CompressedTensor((2, 2, 2), starm.TransformSet((starm.identity_transform(2),)), f,
                               "tsvdm2", 0.5)
    out["cmp_small"] = hexof(starm.write_compressed, c)
    t = starm.DenseTensor(np.random.default_rng(9).standard_normal(5 * 4 * 3 * 2), (5, 4, 3, 2), copy=False)
    ts = starm.TransformSet.build(t.dims, ["data-driven", starm.validate_transform(orthonormal(2, 4))],
                                  tensor=t)
    out["cmp_mixed"] = hexof(starm.write_compressed, starm.tsvdm_tolerance(t, ts, 0.35))
    t = starm.DenseTensor(np.random.default_rng(3).standard_normal(6 * 5 * 8), (6, 5, 8), copy=False)
    out["ten_dct"] = hexof(starm.write_tensor, t)
    ts = starm.TransformSet.build(t.dims, "dct")
    out["cmp_dct"] = hexof(starm.write_compressed, starm.tsvdm_fixed_rank(t, ts, 2))
    with open(os.path.join(HERE, "codec_golden.json"), "w") as fh:
        json.dump(out, fh, indent=0)
    print({k: len(v) // 2 for k, v in out.items()})


if __name__ == "__main__":
    main()
