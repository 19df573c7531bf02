#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gmm_gpu.py -q -x > gpurun_out/pytest_gmm.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gmm.log
timeout 900 python bench.py --workload gmm > gpurun_out/bench_gmm.json 2> gpurun_out/bench_gmm.err; echo "bench gmm rc=$?"
timeout 900 python bench.py --workload gmm_large --steps 3 --warmup 3 --no-e2e > gpurun_out/bench_gmm_large.json 2> gpurun_out/bench_gmm_large.err; echo "bench gmm_large rc=$?"
