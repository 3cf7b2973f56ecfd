"""GPU-backed ``starm`` CLI: exit codes, stdout lines and
file interop, mirroring reference tests/test_cli.py.  Commands that compute
are GPU tests; usage errors, info and error run on the CPU."""

import io
import json
import os

import numpy as np
import pytest

from paper_2605_16058_b200 import DenseTensor, codec
from paper_2605_16058_b200.cli import main

with open(os.path.join(os.path.dirname(__file__), "golden", "codec_golden.json")) as _fh:
    GOLD = {k: bytes.fromhex(v) for k, v in json.load(_fh).items()}


def run(capsys, *argv):
    code = main([str(a) for a in argv])
    cap = capsys.readouterr()
    return code, cap.out, cap.err


def kv(out):
    return dict(line.split("=", 1) for line in out.strip().splitlines())


def test_info_on_reference_artifact(tmp_path, capsys):
    path = tmp_path / "c.cmp"
    path.write_bytes(GOLD["cmp_mixed"])
    code, out, _ = run(capsys, "info", path)
    assert code == 0
    d = kv(out)
    assert d["kind"] == "compressed" and d["dims"] == "5x4x3x2" and d["method"] == "tsvdm2"
    assert d["transforms"] == "data-driven,custom"
    c = codec.read_compressed(path)
    hist = dict(map(int, x.split(":")) for x in d["rank_hist"].split(","))
    assert sum(hist.values()) == c.ranks.size


def test_info_on_tensor(tmp_path, capsys):
    path = tmp_path / "t.ten"
    path.write_bytes(GOLD["ten_dct"])
    code, out, _ = run(capsys, "info", path)
    d = kv(out)
    assert code == 0 and d["kind"] == "tensor" and d["dims"] == "6x5x8"
    assert d["norm"] == format(codec.read_tensor(path).frobenius_norm(), ".6g")


def test_error_command(tmp_path, capsys):
    a = DenseTensor(np.arange(1.0, 25.0), (2, 3, 4))
    b = DenseTensor(np.arange(1.0, 25.0) * 1.5, (2, 3, 4))
    codec.write_tensor(a, tmp_path / "a.ten")
    codec.write_tensor(b, tmp_path / "b.ten")
    code, out, _ = run(capsys, "error", tmp_path / "a.ten", tmp_path / "a.ten")
    assert code == 0 and float(out) == 0.0
    code, out, _ = run(capsys, "error", tmp_path / "a.ten", tmp_path / "b.ten")
    assert code == 0 and out.strip() == format(0.5, ".6g")


def test_usage_errors_exit_two(tmp_path, capsys):
    src = tmp_path / "t.ten"
    src.write_bytes(GOLD["ten_dct"])
    dst = tmp_path / "o.cmp"
    assert run(capsys, "compress", src, dst, "--tol", "1.5")[0] == 2
    assert run(capsys, "compress", src, dst, "--method", "tsvdm1")[0] == 2           # no --rank
    assert run(capsys, "compress", src, dst, "--method", "tsvdm1", "--rank", "2",
               "--tol", "0.1")[0] == 2                                              # both
    assert run(capsys, "compress", tmp_path / "nope.ten", dst, "--tol", "0.1")[0] == 2
    assert run(capsys, "compress", src, dst, "--tol", "0.1", "--transform", "dct,dct")[0] == 2
    assert run(capsys, "badcommand")[0] == 2
    bad = tmp_path / "bad.ten"
    bad.write_bytes(b"XXXXXXXX" + GOLD["ten_dct"][8:])
    for argv in (("info", bad), ("decompress", bad, tmp_path / "o.ten"), ("error", bad, bad)):
        code, _, err = run(capsys, *argv)
        assert code == 2 and "magic" in err


def test_mismatched_dims_exit_two(tmp_path, capsys):
    codec.write_tensor(DenseTensor(np.ones(8), (2, 2, 2)), tmp_path / "a.ten")
    codec.write_tensor(DenseTensor(np.ones(12), (2, 3, 2)), tmp_path / "b.ten")
    code, _, err = run(capsys, "error", tmp_path / "a.ten", tmp_path / "b.ten")
    assert code == 2 and "dims differ" in err


@pytest.mark.gpu
def test_compress_decompress_error_pipeline(tmp_path, capsys):
    import paper_2605_16058_b200 as sb
    src = tmp_path / "a.ten"
    t = DenseTensor(np.random.default_rng(11).standard_normal(7 * 6 * 5 * 2), (7, 6, 5, 2))
    codec.write_tensor(t, src)
    cmp_path = tmp_path / "a.cmp"
    code, out, _ = run(capsys, "compress", src, cmp_path, "--method", "tsvdm2", "--tol", "0.3")
    assert code == 0
    printed = kv(out)
    c = sb.tsvdm_tolerance(t, sb.TransformSet.build(t.dims, "dct"), 0.3)
    assert printed["error"] == format(c.relative_error(), ".6g")
    assert printed["ratio"] == format(sb.compression_ratio(c), ".6g")
    out_path = tmp_path / "b.ten"
    assert run(capsys, "decompress", cmp_path, out_path)[0] == 0
    code, out, _ = run(capsys, "error", src, out_path)
    assert code == 0 and abs(float(out) - c.relative_error()) <= 1e-5 * c.relative_error()
    assert float(out) <= 0.3


@pytest.mark.gpu
def test_compress_fixed_rank_and_reference_decompress_agree(tmp_path, capsys):
    """A GPU-written artifact and the reference's artifact of the same input
    decompress (on the GPU) to the same tensor."""
    src = tmp_path / "t.ten"
    src.write_bytes(GOLD["ten_dct"])
    ours = tmp_path / "ours.cmp"
    code, _, _ = run(capsys, "compress", src, ours, "--method", "tsvdm1", "--rank", "2")
    assert code == 0
    ref = tmp_path / "ref.cmp"
    ref.write_bytes(GOLD["cmp_dct"])
    assert run(capsys, "decompress", ours, tmp_path / "a.ten")[0] == 0
    assert run(capsys, "decompress", ref, tmp_path / "b.ten")[0] == 0
    code, out, _ = run(capsys, "error", tmp_path / "b.ten", tmp_path / "a.ten")
    assert code == 0 and float(out) <= 1e-10
    code, out, _ = run(capsys, "info", ours)
    assert kv(out)["rank_hist"] == "2:8"


@pytest.mark.gpu
def test_gen_and_bench_csv(tmp_path, capsys):
    path = tmp_path / "g.ten"
    assert run(capsys, "gen", path, "--dims", "6,5,4", "--seed", "3")[0] == 0
    assert codec.read_tensor(path).dims == (6, 5, 4)
    csv_path = tmp_path / "b.csv"
    code, out, _ = run(capsys, "bench", "--kernel", "tsvdm2", "--input", path, "--trials", "2",
                       "--csv", csv_path)
    assert code == 0 and "median=" in out
    lines = csv_path.read_text().strip().splitlines()
    assert lines[0] == ",".join(codec.CSV_FIELDS) and len(lines) == 1 + 3 * 2
