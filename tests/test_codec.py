"""File formats: byte-identical .ten / .cmp against bytes
the reference package wrote (tests/golden/make_codec_golden.py), the error
taxonomy of reference tests/test_codec.py, and GPU results written through
the same writer."""

import csv
import io
import json
import os
import struct

import numpy as np
import pytest

from paper_2605_16058_b200 import (CompressedTensor, DenseTensor, TransformSet, VariableRankFactors,
                                   identity_transform)
from paper_2605_16058_b200 import codec
from paper_2605_16058_b200.codec import (BadMagicError, FormatError, TruncatedPayloadError,
                                         UnsupportedDtypeError, UnsupportedVersionError)

with open(os.path.join(os.path.dirname(__file__), "golden", "codec_golden.json")) as _fh:
    GOLD = {k: bytes.fromhex(v) for k, v in json.load(_fh).items()}


def small_compressed():
    f = VariableRankFactors(2, 2, np.array([1, 0]), np.array([1.0, 2.0]), np.array([3.0, 4.0]))
    return CompressedTensor((2, 2, 2), TransformSet((identity_transform(2),)), f, "tsvdm2", 0.5)


def written(writer, obj):
    buf = io.BytesIO()
    writer(obj, buf)
    return buf.getvalue()


def test_golden_bytes_small():
    t = DenseTensor(np.arange(8.0), (2, 2, 2), copy=False)
    assert written(codec.write_tensor, t) == GOLD["ten_small"]
    assert len(GOLD["ten_small"]) == 38 + 64
    assert written(codec.write_compressed, small_compressed()) == GOLD["cmp_small"]


@pytest.mark.parametrize("key", ["cmp_small", "cmp_mixed", "cmp_dct"])
def test_reference_artifacts_round_trip_bitwise(key):
    c = codec.read_compressed(io.BytesIO(GOLD[key]))
    assert written(codec.write_compressed, c) == GOLD[key]
    assert c.relative_error() is None  # energies are not stored


@pytest.mark.parametrize("key", ["ten_small", "ten_dct"])
def test_reference_tensors_round_trip_bitwise(key, tmp_path):
    t = codec.read_tensor(io.BytesIO(GOLD[key]))
    path = tmp_path / "t.ten"
    codec.write_tensor(t, path)
    assert path.read_bytes() == GOLD[key]
    assert codec.read_tensor(path).dims == t.dims


def test_mixed_artifact_fields():
    c = codec.read_compressed(io.BytesIO(GOLD["cmp_mixed"]))
    assert c.dims == (5, 4, 3, 2)
    assert c.method == "tsvdm2" and c.param == 0.35
    assert c.transforms.kinds == ("data-driven", "custom")
    assert c.factors.u_data.size == c.ranks.sum() * 5
    assert c.factors.g_data.size == c.ranks.sum() * 4


def test_zero_ranks_round_trip():
    back = codec.read_compressed(io.BytesIO(GOLD["cmp_small"]))
    assert list(back.ranks) == [1, 0]
    assert back.factors.u_block(1).shape == (2, 0)


def test_tensor_error_taxonomy():
    good = bytearray(GOLD["ten_small"])
    for pos, val, exc in ((0, ord("X"), BadMagicError), (8, 9, UnsupportedVersionError),
                          (9, 7, UnsupportedDtypeError), (14, 0, FormatError)):
        bad = good.copy()
        bad[pos] = val
        with pytest.raises(exc):
            codec.read_tensor(io.BytesIO(bytes(bad)))
    for cut in (4, 12, 30, 38, 70, len(good) - 1):
        with pytest.raises(TruncatedPayloadError):
            codec.read_tensor(io.BytesIO(bytes(good[:cut])))


def test_compressed_error_taxonomy():
    good = bytearray(GOLD["cmp_small"])
    cases = ((7, ord("X"), BadMagicError), (8, 2, UnsupportedVersionError), (9, 99, FormatError),
             (46, 250, FormatError),  # transform kind byte
             (47, 9, FormatError),    # slice count no longer matches dims
             (55, 3, FormatError),    # rank above min(m, p)
             (9, 1, FormatError))     # fixed-rank method with ranks (1, 0): not uniform
    for pos, val, exc in cases:
        bad = good.copy()
        bad[pos] = val
        with pytest.raises(exc):
            codec.read_compressed(io.BytesIO(bytes(bad)))
    for cut in (6, 20, 40, 50, 60, len(good) - 4):
        with pytest.raises(TruncatedPayloadError):
            codec.read_compressed(io.BytesIO(bytes(good[:cut])))


def test_broken_stored_transform_rejected():
    raw = bytearray(GOLD["cmp_mixed"])
    offset = 8 + 14 + 4 * 8 + 2 + 8 + 4 * 6  # first stored matrix entry (mode-2 data-driven)
    raw[offset:offset + 8] = np.array([7.5]).tobytes()
    with pytest.raises(FormatError):
        codec.read_compressed(io.BytesIO(bytes(raw)))


def test_huge_declaration_fails_before_allocating(tmp_path):
    body = b"STARMTEN" + struct.pack("<BBI", 1, 0, 3) + np.asarray([1000] * 3, dtype="<u8").tobytes()
    path = tmp_path / "huge.ten"
    path.write_bytes(body + b"\x00" * 16)  # 8 GB declared, 16 bytes present
    with pytest.raises(TruncatedPayloadError):
        codec.read_tensor(path)


def test_max_mode_count():
    with pytest.raises(FormatError):
        codec.read_tensor(io.BytesIO(b"STARMTEN" + struct.pack("<BBI", 1, 0, 4_000_000)))


def test_bench_csv_schema(tmp_path):
    rows = [codec.BenchRow("ttm", "batched", "2", 1, 0, 0.00125, 4096),
            codec.BenchRow("svd", "slices-parallel", "", 4, 1, 0.5, 123456)]
    path = tmp_path / "bench.csv"
    codec.write_bench_csv(rows, path)
    with open(path, newline="") as fh:
        parsed = list(csv.reader(fh))
    assert parsed[0] == list(codec.CSV_FIELDS) and len(parsed) == 3
    assert float(parsed[1][5]) == 0.00125 and int(parsed[2][6]) == 123456


# ------------------------------------------------------------ GPU results

@pytest.mark.gpu
def test_gpu_artifact_interoperates_with_reference_artifact():
    """Compress the reference's own input on the GPU, write it, and check the
    header + ranks bytes equal the reference's artifact and both artifacts
    reconstruct the same tensor (U/V signs are free, so payload bytes are
    compared through the reconstruction)."""
    import paper_2605_16058_b200 as sb
    t = codec.read_tensor(io.BytesIO(GOLD["ten_dct"]))
    ts = sb.TransformSet.build(t.dims, "dct")
    ours = written(codec.write_compressed, sb.tsvdm_fixed_rank(t, ts, 2))
    ref = GOLD["cmp_dct"]
    head = 8 + 14 + 3 * 8 + 1 + 8 + 4 * 8  # through the ranks
    assert len(ours) == len(ref) and ours[:head] == ref[:head]
    rec_ours = sb.reconstruct(codec.read_compressed(io.BytesIO(ours))).data
    rec_ref = sb.reconstruct(codec.read_compressed(io.BytesIO(ref))).data
    assert np.linalg.norm(rec_ours - rec_ref) <= 1e-10 * np.linalg.norm(rec_ref)


@pytest.mark.gpu
def test_device_results_write_like_host_results():
    import torch
    import paper_2605_16058_b200 as sb
    t = codec.read_tensor(io.BytesIO(GOLD["ten_dct"]))
    x = sb.DeviceTensor.from_host(t, torch.device("cuda", 0))
    assert written(codec.write_tensor, x) == GOLD["ten_dct"]
    ts = sb.TransformSet.build(t.dims, "dct")
    c_dev = sb.tsvdm_tolerance(x, ts, 0.3)      # DeviceFactors
    assert written(codec.write_compressed, c_dev) == written(codec.write_compressed, c_dev.to_host())
