#!/bin/bash
# One gpurun call: GPU tests, bench lines, launch lists, full ncu captures.
# Every ncu command re-runs a command line that has just exited 0 without ncu.
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvidia-smi.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
timeout 600 python bench.py --workload ba > gpurun_out/bench_ba.json 2> gpurun_out/bench_ba.err; echo "bench ba rc=$?"
SMALL="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --n 16777216"
BA="python bench.py --workload ba --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
if [ "${NO_NCU:-0}" = "1" ]; then exit 0; fi
timeout 300 $SMALL > gpurun_out/bench_small.json 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_bessel.csv $SMALL > gpurun_out/ncu_launches.log 2>&1
echo "launches rc=$?"
timeout 300 $SMALL > /dev/null 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_besselj -s 3 -c 1 \
    -o gpurun_out/prof_bessel $SMALL > gpurun_out/ncu_full.log 2>&1
echo "full rc=$?"
timeout 300 $BA > gpurun_out/bench_ba_small.json 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_ba.csv $BA > gpurun_out/ncu_launches_ba.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_ba_jac -s 3 -c 1 \
    -o gpurun_out/prof_ba $BA > gpurun_out/ncu_full_ba.log 2>&1
echo "ba ncu rc=$?"
