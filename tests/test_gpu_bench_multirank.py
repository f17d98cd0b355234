"""GPU: bench.py's multi-rank path (torch.distributed.run, 2 ranks) end to end on the one GPU of
this box — both ranks on cuda:0 with the gloo backend (CB_BENCH_SHARE_GPU / CB_BENCH_BACKEND;
host barriers only, no kernel waits on the other rank).  Checks the JSON contract of an N > 1
line (n_gpus, strong scaling over one M batch, max-over-ranks timing, parallelism text), not
its numbers (two ranks sharing one GPU are not a scaling measurement)."""

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


@pytest.mark.parametrize("cfg", ["2", "3"])
def test_bench_two_ranks_one_gpu(cuda, cfg):
    env = dict(os.environ, CB_BENCH_SHARE_GPU="1", CB_BENCH_BACKEND="gloo")
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK"):
        env.pop(k, None)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2", "--master-addr",
           "127.0.0.1", "--master-port", str(_port()), os.path.join(ROOT, "bench.py"), "--gpus", "2", "--config", cfg,
           "--steps", "1", "--warmup", "3"]
    p = subprocess.run(cmd, capture_output=True, text=True, env=env, timeout=600, cwd=ROOT)
    assert p.returncode == 0, p.stderr[-2000:]
    lines = [ln for ln in p.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, p.stdout[-2000:]   # rank 0 prints the one line
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["scaling"] == "strong"
    assert d["cpu_baseline"] is None           # CPU baseline only at N = 1
    assert ("dp2" in d["config"]["parallelism"]) or ("node-shard2" in d["config"]["parallelism"])
