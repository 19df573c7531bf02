"""The N > 1 bench path end to end on the device: two ranks (both folded
onto the visible GPU, gloo for the plumbing: `--dist-backend gloo`) run the
sharded Bessel / BA / GMM steps, the GMM all_reduce of the packed shard
gradients, the max-over-ranks timing and the shard host entries of the e2e
numbers.  Timings are meaningless here (two ranks share one GPU); the line's
shape and the sharded results' consistency are what is checked."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_two_ranks_on_one_gpu_over_gloo():
    out = subprocess.run(
        [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
         "--master-addr", "127.0.0.1", "--master-port", "29517", os.path.join(REPO, "bench.py"),
         "--gpus", "2", "--dist-backend", "gloo", "--steps", "3", "--warmup", "3",
         "--no-cpu-baseline"],
        capture_output=True, text=True, timeout=900, cwd=REPO)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1                                  # rank 0 alone prints
    r = json.loads(lines[0])
    assert r["n_gpus"] == 2 and r["dist"]["world_size"] == 2
    for sub in (r, r["ba"], r["gmm_c3"], r["gmm_c5"]):
        assert sub["n_gpus"] == 2 and sub["value"] > 0 and sub["e2e"]["value"] > 0
        assert sub["failed_per_step"] == 0
    assert "shard" in r["gmm_c3"]["e2e"]["path"]
