"""bench.py's multi-rank flow (torchrun, one process per rank, max over ranks, per-rank times)
run on the one GPU gpurun gives: two gloo ranks share cuda:0 (B200RT_SHARE_GPU=1). Their
kernels never wait on each other's, so this checks the launch, the collective's plumbing and
the JSON line, not scaling; the benchmark itself runs NCCL with one GPU per rank."""
import json
import os
import socket
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.gpu
def test_bench_two_ranks_share_one_gpu():
    env = dict(os.environ, B200RT_DIST_BACKEND="gloo", B200RT_SHARE_GPU="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2", "--master-addr",
           "127.0.0.1", "--master-port", str(_free_port()), "bench.py", "--gpus", "2", "--config", "C2", "--steps",
           "3", "--warmup", "1", "--no-cpu-baseline", "--no-fp32-peak"]
    out = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]  # rank 0 alone prints
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["steps"] == 3 and d["value"] > 0
    assert d["warmup"] == 3  # at least 3 warm-up steps run (and are reported) whatever --warmup says
    assert d["config"]["workload"] == "C2" and d["config"]["parallelism"] == "tiles2"
    pr = d["per_rank"]
    assert len(pr["step_ms"]) == 2 and len(pr["shard_render_ms"]) == 2
    assert all(x > 0 for x in pr["step_ms"]) and all(x > 0 for x in pr["shard_render_ms"])
    assert d["e2e"]["value"] > 0 and d["gpu_launches"] > 0
