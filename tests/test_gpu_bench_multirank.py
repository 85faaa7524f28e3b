"""bench.py's multi-rank path (torchrun, N > 1) end to end on the one lease GPU: two ranks share
cuda:0 over gloo (SPA2_BENCH_BACKEND=gloo; NCCL needs one GPU per rank), so the code the driver's
multi-GPU bench runs — batch-sharded weak scaling, max-over-ranks timing, the configs[3] leg with
head sharding + all-gather and the overlapped Ulysses operator — executes and prints one JSON line
with the cfg4 results.  The timings of two ranks time-sharing one GPU are meaningless."""

import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_bench_two_ranks_one_gpu():
    env = {**os.environ, "SPA2_BENCH_BACKEND": "gloo"}
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2", "--master-addr",
           "127.0.0.1", "--master-port", str(_free_port()), os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps",
           "3", "--warmup", "3", "--no-e2e", "--ulysses-groups", "2"]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=1200)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-6000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["n_gpus"] == 2 and line["value"] > 0
    c4 = line["cfg4"]
    assert c4["heads_per_rank"] == 20
    assert c4["head_sharded"]["ms_per_step"] > 0 and c4["head_sharded"]["allgather_ms_per_step"] > 0
    assert c4["ulysses"]["ms_per_step"] > 0 and c4["ulysses"]["alltoall_ms_per_step"] > 0
