"""bench.py's driver contract on the CPU side: the reference arm prints one
JSON line with the contract keys (every workload), under torchrun only rank 0
prints, and the ours-arm line builders produce the required keys (checked on
the GPU by the bench itself)."""

import json
import os
import subprocess
import sys

import pytest

from conftest import REPO

KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
        "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config", "impl",
        "cpu_baseline", "e2e"}


def run_bench(*args, env=None, timeout=240):
    e = dict(os.environ, **(env or {}))
    out = subprocess.run([sys.executable, os.path.join(REPO, "bench.py"), *args],
                         capture_output=True, text=True, timeout=timeout, env=e, cwd=REPO)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.strip().startswith("{")]
    return [json.loads(ln) for ln in lines]


@pytest.mark.parametrize("workload", ["bessel", "ba", "gmm_large"])
def test_reference_arm_line(workload):
    (line,) = run_bench("--impl", "reference", "--workload", workload, "--steps", "2",
                        "--warmup", "1")
    if "unavailable" in line:
        assert workload == "gmm_large" and line["impl"] == "reference"
        return
    assert KEYS <= set(line), KEYS - set(line)
    assert line["impl"] == "reference" and line["value"] > 0
    assert line["cpu_baseline"]["kind"] == "port" and line["cpu_baseline"]["cores"] >= 1
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["value"] == line["value"]
    assert line["config"]["workload"]


def test_reference_arm_under_torchrun_prints_once():
    out = subprocess.run(
        [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
         "--master-addr", "127.0.0.1", "--master-port", "29611", os.path.join(REPO, "bench.py"),
         "--impl", "reference", "--steps", "1", "--warmup", "1"],
        capture_output=True, text=True, timeout=300, cwd=REPO)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.strip().startswith("{")]
    assert len(lines) == 1
    line = json.loads(lines[0])
    assert line["cpu_baseline"]["cores"] == (os.cpu_count() or 1)   # all host threads
