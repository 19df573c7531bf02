#!/bin/bash
mkdir -p gpurun_out
SMALL="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --n 16777216"
timeout 300 $SMALL > gpurun_out/bench_small.json 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_besselj -s 3 -c 1 \
    -o gpurun_out/prof_bessel $SMALL > gpurun_out/ncu_full.log 2>&1
echo "full rc=$?"
