"""bench.py's N > 1 path end to end: two ranks under torchrun, each sweeping
its column shard of the C2-distributed matrix, the per-iteration exchange
through a gloo group (GPSPCA_BENCH_BACKEND=gloo: with one GPU the ranks share
it, so the peer-memory kernel -- whose ranks spin on each other -- must not
run; timings are meaningless here).  Checks that rank 0 prints one JSON line
with n_gpus = 2, the exchange path named, and the sharded loop reaching
every timed iteration."""

import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_bench_two_ranks_gloo():
    pytest.importorskip("torch")
    env = dict(os.environ, GPSPCA_BENCH_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes", "1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), "bench.py", "--gpus", "2",
           "--steps", "4", "--warmup", "3", "--cols", str(1 << 18), "--no-block", "--e2e-steps", "3",
           "--no-cpu-baseline"]
    out = subprocess.run(cmd, capture_output=True, text=True, cwd=ROOT, env=env, timeout=600)
    assert out.returncode == 0, out.stdout[-3000:] + out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout[-3000:]
    rec = json.loads(lines[0])
    assert rec["n_gpus"] == 2 and rec["steps"] == 4 and rec["warmup"] == 3
    assert rec["config"]["exchange"] == "torch.distributed all_reduce (gloo)"
    assert rec["config"]["parallelism"] == "column-shard x2"
    assert rec["value"] > 0 and rec["gpu_launches"] > 0
    assert rec["e2e"]["value"] > 0 and rec["e2e"]["steps"] == 3 and rec["e2e"]["h2d_bytes_per_step"] > 0
