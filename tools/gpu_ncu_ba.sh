#!/bin/bash
mkdir -p gpurun_out
BA="python bench.py --workload ba --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 300 $BA > gpurun_out/bench_ba_small.json 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_ba_jac -s 3 -c 1 \
    -o gpurun_out/prof_ba $BA > gpurun_out/ncu_full_ba.log 2>&1
echo "ba ncu rc=$?"
