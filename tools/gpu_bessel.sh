#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_bessel_gpu.py tests/test_run_gpu.py -q -x > gpurun_out/pytest_bessel.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_bessel.log
timeout 600 python bench.py --no-e2e --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
