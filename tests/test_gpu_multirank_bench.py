"""The bench's N > 1 code path on the one-GPU box (bench.py):
two ranks launched by torch.distributed.run share cuda:0 with the collectives
over gloo (SD_BENCH_SHARED_GPU=1).  Samples are sharded by global id, each
rank runs its own device loop, the timing is the max over ranks and rank 0
alone prints one JSON line for the whole job.  Run on C2 (small) so it takes
seconds; the numbers are not measurements (two ranks share one GPU)."""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_two_ranks_share_one_gpu_and_rank0_prints_one_line():
    env = dict(os.environ, SD_BENCH_SHARED_GPU="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(free_port()), os.path.join(ROOT, "bench.py"),
           "--config", "c2", "--gpus", "2", "--steps", "1", "--warmup", "1", "--no-cpu", "--max-new", "32"]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2
    assert d["config"]["global_batch"] == 16 and d["config"]["batch_per_gpu"] == 8
    assert d["value"] > 0 and d["padded"]["value"] > 0
    assert d["scaling"] == "weak"
