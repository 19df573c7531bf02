#!/bin/bash
mkdir -p gpurun_out
G="python bench.py --workload gmm_large --n 100000 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 600 $G > gpurun_out/bench_gmm_mid.json 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_gmm_large.csv $G > gpurun_out/ncu_launches_gmm.log 2>&1 && \
  timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"k_gmm_(fwd|rev|lse)" -s 6 -c 3 \
    -o gpurun_out/prof_gmm_large $G > gpurun_out/ncu_full_gmm_large.log 2>&1
echo "rc=$?"
