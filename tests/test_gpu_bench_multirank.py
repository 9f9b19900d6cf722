"""bench.py's N > 1 path (the driver's scaling run) end to end: two ranks under torch.distributed.run,
gloo on the one GPU (RLK_BENCH_BACKEND=gloo; NCCL refuses two ranks per GPU) -- sharded fusion with
the compact partials all-reduce, the rank-partitioned e2e stream and the sharded GRPO loss, max over
ranks, one JSON line from rank 0."""
import json
import os
import socket
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_bench_two_ranks(cuda):
    env = dict(os.environ, RLK_BENCH_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), "bench.py", "--gpus", "2", "--steps", "2",
           "--warmup", "3", "--quick", "--no-cpu", "--layout", "gpt1p3b", "--grpo-tokens", "4096",
           "--e2e-budget-gb", "8"]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, (r.stdout + r.stderr)[-4000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]  # rank 0 alone prints
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["e2e"]["value"] > 0 and d["grpo"]["tokens_per_s"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] == d["config"]["params"] * 2 * 4
