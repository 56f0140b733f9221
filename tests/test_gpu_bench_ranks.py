"""The N > 1 path of bench.py (sharded population, per-generation elite
all-gather, max-over-ranks timing) run as two ranks on one GPU over gloo --
the box has a single GPU, so NCCL itself is exercised only at N = 1."""

import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_two_rank_bench_line(gpu):
    env = dict(os.environ, CB_BENCH_DIST_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), "bench.py", "--gpus", "2",
           "--workload", "bert_base", "--steps", "3", "--warmup", "3", "--population", "262144", "--search-generations", "3",
           "--e2e-steps", "1"]
    out = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1  # rank 0 alone prints
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["config"]["global_population"] == 2 * 262144
    assert d["value"] > 0 and d["e2e"]["value"] > 0
    assert d["search"]["best_cost_ms_after_timed_steps"] <= d["search"]["dp_cost_ms"]
    assert "configs" not in d and "cpu_baseline" not in d  # rank-0, N = 1 extras only
