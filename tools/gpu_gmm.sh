#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gmm_gpu.py tests/test_run_gpu.py -q -x > gpurun_out/pytest_gmm.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gmm.log
timeout 600 python bench.py --workload gmm --no-e2e --no-cpu-baseline > gpurun_out/bench_gmm.json 2> gpurun_out/bench_gmm.err; echo "bench rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_gmm.csv python bench.py --workload gmm --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launches_gmm.log 2>&1; echo "launches rc=$?"
