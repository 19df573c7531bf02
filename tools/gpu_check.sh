#!/bin/bash
# One gpurun call: GPU tests, bench, launch list, full ncu capture of the top
# kernel, FP64 weights.  Every ncu command re-runs a command that has just
# exited 0 without ncu.
set -x
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvidia-smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
SMALL="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --n 16777216"
timeout 300 $SMALL > gpurun_out/bench_small.json 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches.csv $SMALL > gpurun_out/ncu_launches.log 2>&1
echo "launches rc=$?"
timeout 300 python tools/probe_weights.py > gpurun_out/probe_plain.log 2>&1 && \
  timeout 600 ncu --metrics sm__sass_thread_inst_executed_op_dfma_pred_on.sum,sm__sass_thread_inst_executed_op_dadd_pred_on.sum,sm__sass_thread_inst_executed_op_dmul_pred_on.sum \
    -k regex:k_unary --csv --log-file gpurun_out/weights.csv python tools/probe_weights.py > gpurun_out/ncu_weights.log 2>&1
echo "weights rc=$?"
timeout 300 $SMALL > /dev/null 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_besselj -s 3 -c 1 \
    -o gpurun_out/prof_bessel $SMALL > gpurun_out/ncu_full.log 2>&1
echo "full rc=$?"
