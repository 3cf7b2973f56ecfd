"""bench.py's multi-GPU launch plumbing on CPU: ``--gpus N`` relaunches under
torch.distributed.run with N ranks (gloo in --dry-run), every rank joins, and
the sharded plan covers every fibre and slice exactly once."""

import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("gpus,config", [(2, "c2"), (4, "c5")])
def test_bench_gpus_n_launches_n_ranks(gpus, config):
    env = dict(os.environ, NCCL_DEBUG="WARN")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", str(gpus),
                          "--config", config, "--dry-run"], capture_output=True, text=True,
                         timeout=240, env=env, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout
    rec = json.loads(lines[0])
    dims = {"c2": (361, 720, 1024), "c5": (8192, 64, 4096)}[config]
    assert rec["world_size"] == gpus and rec["mode"] == "sharded"
    assert rec["fibres"] == dims[0] * dims[1] and rec["slices"] == dims[2]
