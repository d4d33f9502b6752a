"""bench.py's row-sharded multi-rank path end to end under
torchrun with 2 ranks.  This box has one GPU, so both ranks share cuda:0 and
the process group uses gloo (test hooks GQSA_SHARE_DEVICE / GQSA_DIST_BACKEND);
the numbers are meaningless, the plumbing (shard packing, per-rank launches,
all-gather, max-over-ranks timing, one JSON line from rank 0) is not."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bench_two_ranks_one_json_line():
    env = dict(os.environ, GQSA_SHARE_DEVICE="1", GQSA_DIST_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", "29623", "bench.py", "--gpus", "2",
           "--steps", "50", "--warmup", "3"]
    out = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["config"]["parallelism"] == "rowshard2" and d["value"] > 0
    assert d["scaling"] == "strong" and d["gpu_launches"] > 0
    mg = d["multi_gpu"]  # kernels and exchange reported apart
    assert mg["per_rank_kernel_us"] > 0 and mg["allgather_us"] > 0 and mg["kernel_only_aggregate_gbs"] > 0
