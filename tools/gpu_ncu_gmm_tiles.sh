#!/bin/bash
mkdir -p gpurun_out
GMM="python bench.py --workload gmm --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 300 $GMM > gpurun_out/bench_gmm_small.json 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_gmm_(fwd|rev)" -s 6 -c 2 \
    -o gpurun_out/prof_gmm_tiles $GMM > gpurun_out/ncu_gmm_tiles.log 2>&1
echo "ncu rc=$?"
