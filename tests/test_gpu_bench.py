"""bench.py end to end at a small scale: the single-GPU line and the N = 2
pipelines (key-partitioned, and the file-sharded hybrid; two ranks sharing
the GPU over gloo) all produce a well-formed JSON line with the contract's
keys."""

from __future__ import annotations

import json
import os
import socket
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parent.parent


def _line(out: str) -> dict:
    lines = [ln for ln in out.splitlines() if ln.startswith("{")]
    assert lines, out[-2000:]
    return json.loads(lines[-1])


def _check(d: dict, n_gpus: int):
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "dtype", "data", "config", "roofline", "e2e", "gpu_launches", "clocks"):
        assert k in d, k
    assert d["n_gpus"] == n_gpus and d["value"] > 0 and d["gpu_launches"] > 0
    assert 0 < d["roofline"]["frac"] < 1.5
    assert d["e2e"]["h2d_bytes_per_step"] > 0


def test_bench_single_gpu_small():
    r = subprocess.run([sys.executable, "bench.py", "--steps", "2", "--warmup", "1", "--scale", "0.05",
                        "--no-cpu-baseline"], cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    _check(_line(r.stdout), 1)


@pytest.mark.parametrize("multi", ["partitioned", "hybrid"])
def test_bench_sharded_two_ranks_small(multi):
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    env = dict(os.environ, MX_BENCH_BACKEND="gloo", MX_BENCH_MULTI=multi)
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                        "--master-addr", "127.0.0.1", "--master-port", str(port), "bench.py", "--gpus", "2",
                        "--steps", "2", "--warmup", "1", "--scale", "0.05"], cwd=ROOT, capture_output=True,
                       text=True, timeout=900, env=env)
    assert r.returncode == 0, r.stderr[-3000:]
    d = _line(r.stdout)
    _check(d, 2)
    assert d["config"]["parallelism"] == ("file-sharded hybrid x2" if multi == "hybrid" else "key-partitioned x2")
    assert d["job"]["chunks"] > 0
