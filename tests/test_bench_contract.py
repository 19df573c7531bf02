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
         "--gpus", "2", "--impl", "reference", "--steps", "1", "--warmup", "1"],
        capture_output=True, text=True, timeout=300, cwd=REPO)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.strip().startswith("{")]
    assert len(lines) == 1
    line = json.loads(lines[0])
    assert line["cpu_baseline"]["cores"] == (os.cpu_count() or 1)   # all host threads


def test_gpus_flag_self_launches_the_ranks():
    """--gpus 2 outside torchrun re-launches bench.py under
    torch.distributed.run with two ranks (gloo dry run: the launch, the
    world-size check and the max-over-ranks timing, no kernels)."""
    (line,) = run_bench("--gpus", "2", "--dry-run", "--steps", "2", "--warmup", "1")
    assert line["n_gpus"] == 2 and line["ranks_reporting"] == 2 and line["dry_run"]
    assert line["dist"]["world_size"] == 2
    assert line["config"]["parallelism"] == "shard2"
    assert line["ms_per_step"] >= 2e-3                 # the max over ranks (rank 1 adds 2e-3)


def test_gpus_one_is_a_single_process():
    (line,) = run_bench("--gpus", "1", "--dry-run", "--steps", "2")
    assert line["n_gpus"] == 1 and line["ranks_reporting"] == 1 and line["dist"] is None


def test_world_size_mismatch_is_an_error():
    out = subprocess.run([sys.executable, os.path.join(REPO, "bench.py"), "--gpus", "4",
                          "--dry-run"], capture_output=True, text=True, timeout=120, cwd=REPO,
                         env=dict(os.environ, WORLD_SIZE="2", RANK="0", LOCAL_RANK="0"))
    assert out.returncode == 2 and "WORLD_SIZE" in out.stderr
    assert not [ln for ln in out.stdout.splitlines() if ln.startswith("{")]


def test_reference_arm_self_launch_and_same_configs():
    """--gpus 2 --impl reference: rank 0 alone prints, with the config dicts
    the ours arm builds for the same launch (bench.bessel_config etc.)."""
    (line,) = run_bench("--gpus", "2", "--impl", "reference", "--steps", "1", "--warmup", "1",
                        timeout=400)
    import importlib.util
    spec = importlib.util.spec_from_file_location("bench", os.path.join(REPO, "bench.py"))
    bench = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(bench)
    assert line["rate_sample"] is True and line["n_gpus"] == 2
    assert line["config"] == bench.bessel_config(bench.BESSEL_N, 2)
    assert line["ba"]["config"] == bench.ba_config(bench.BA_P, 2)
    assert line["gmm_c3"]["config"] == bench.gmm_config(64, 25, 10000, 2)
    assert line["gmm_c5"]["config"] == bench.gmm_config(128, 200, 1000000, 2)
    for k in ("ba", "gmm_c3", "gmm_c5"):
        assert KEYS <= set(line[k]), KEYS - set(line[k])
