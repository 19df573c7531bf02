#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_ba_gpu.py tests/test_ba_csr_gpu.py tests/test_run_gpu.py -q -x > gpurun_out/pytest_ba.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_ba.log
timeout 600 python bench.py --workload ba --no-e2e --no-cpu-baseline > gpurun_out/bench_ba.json 2> gpurun_out/bench_ba.err; echo "bench rc=$?"
