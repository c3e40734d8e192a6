"""bench.py's N > 1 path on a one-GPU box: two ranks over gloo on GPU 0
(`--dist-backend gloo`, a functional check: strong-scaled sharding through
dist.Sharder, the chunked all-gather, max-over-ranks timing, rank-0 JSON).
The NCCL path needs >= 2 GPUs (tests/test_gpu_dist.py)."""
import json
import os
import socket
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("workload,scale", [("cfg3", "0.02"), ("cfg2", "0.01"), ("cfg5", "0.005")])
def test_bench_two_ranks_gloo(workload, scale):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), os.path.join(ROOT, "bench.py"),
           "--gpus", "2", "--dist-backend", "gloo", "--steps", "3", "--warmup", "3", "--workload", workload,
           "--scale", scale, "--no-cpu-baseline", "--e2e-steps", "1"]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1  # rank 0 only
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["scaling"] == "strong" and d["value"] > 0
    sh = d["config"]["sharding"]
    assert sh["allgather_chunks"] == 2 and sh["pairs_total"] > sh["pairs_this_rank"] > 0
