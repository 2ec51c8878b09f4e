"""bench.py's driver contract on the GPU: one JSON line with the required keys, at N=1 and as a
torchrun world of 2 (both ranks on the box's one GPU, gloo for the timing collective -- the
driver's N>1 runs use NCCL over distinct GPUs), for our arm and the reference arm."""

import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
        "vs_baseline", "dtype", "data", "config", "e2e", "roofline", "clocks", "gpu_launches"}


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _run(args, world=1, env=None):
    e = dict(os.environ, **(env or {}))
    if world > 1:
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
               "--master-addr", "127.0.0.1", f"--master-port={_port()}", "bench.py", "--gpus", str(world)] + args
        e["MF_DIST_BACKEND"] = "gloo"
    else:
        cmd = [sys.executable, "bench.py"] + args
    p = subprocess.run(cmd, cwd=ROOT, env=e, capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stderr[-3000:]
    lines = [ln for ln in p.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, p.stdout[-3000:]
    return json.loads(lines[0])


def test_bench_line_single_gpu():
    d = _run(["--config", "cfg1", "--steps", "3", "--warmup", "3", "--no-cpu-baseline"])
    assert KEYS <= set(d), KEYS - set(d)
    assert d["n_gpus"] == 1 and d["steps"] == 3 and d["warmup"] == 3
    assert d["value"] > 0 and d["e2e"]["value"] > 0 and d["gpu_launches"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0
    assert 0 < d["roofline"]["frac"] < 1


def test_bench_line_world2():
    d = _run(["--config", "cfg4", "--steps", "3", "--warmup", "3", "--no-cpu-baseline"], world=2)
    assert KEYS <= set(d), KEYS - set(d)
    assert d["n_gpus"] == 2 and d["scaling"] == "strong"  # cfg4: one batch sharded
    assert d["value"] > 0 and d["e2e"]["value"] > 0


def test_reference_arm_world2():
    d = _run(["--config", "cfg1", "--steps", "1", "--warmup", "1", "--impl", "reference"], world=2)
    assert d["impl"] == "reference" and d["value"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["cpu_baseline"]["kind"] in ("port", "reference")
