"""The bench's N > 1 code path on a GPU box with one GPU: two ranks share GPU 0
over gloo (PICKER_BENCH_SHARE_GPU=1; NCCL needs one GPU per rank).  Each rank
generates its shard on the GPU (K6), validates it in chunks whose bit-mask
all-gathers overlap the next chunk (dist.ChunkedExchange, CUDA streams), and
rank 0 reports parity of both shards against the tiled oracle codes and the
global histogram."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bench_two_ranks_one_gpu():
    env = dict(os.environ, PICKER_BENCH_SHARE_GPU="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", "29533", os.path.join(ROOT, "bench.py"), "--gpus", "2",
           "--steps", "2", "--warmup", "3", "--replicas", "8", "--no-cpu-baseline", "--no-latency",
           "--e2e-steps", "1", "--chunks", "3"]
    r = subprocess.run(cmd, capture_output=True, text=True, env=env, cwd=ROOT, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["n_gpus"] == 2
    assert line["parity"]["mismatches"] == 0
    assert sum(line["verdict_counts"]) == line["config"]["records_total"] == 2 * 8 * 18217
