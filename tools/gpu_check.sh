#!/bin/bash
# One gpurun call: GPU tests, bench lines, probes; ncu captures unless NO_NCU=1.
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvidia-smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
timeout 600 python bench.py --workload ba > gpurun_out/bench_ba.json 2> gpurun_out/bench_ba.err; echo "bench ba rc=$?"
timeout 900 python bench.py --workload gmm > gpurun_out/bench_gmm.json 2> gpurun_out/bench_gmm.err; echo "bench gmm rc=$?"
timeout 900 python bench.py --workload gmm_large --steps 3 --warmup 3 --no-e2e > gpurun_out/bench_gmm_large.json 2> gpurun_out/bench_gmm_large.err; echo "bench gmm_large rc=$?"
timeout 300 python tools/probe_weights.py > gpurun_out/probe_plain.log 2>&1
if [ "${NO_NCU:-0}" = "1" ]; then exit 0; fi
SMALL="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
BA="python bench.py --workload ba --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
GMM="python bench.py --workload gmm --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 300 $SMALL > gpurun_out/bench_small.json 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_besselj -s 3 -c 1 \
    -o gpurun_out/prof_bessel $SMALL > gpurun_out/ncu_full.log 2>&1
echo "bessel ncu rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_bessel.csv $SMALL > gpurun_out/ncu_launches_bessel.log 2>&1
echo "bessel launches rc=$?"
timeout 300 $BA > gpurun_out/bench_ba_small.json 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_ba_jac -s 3 -c 1 \
    -o gpurun_out/prof_ba $BA > gpurun_out/ncu_full_ba.log 2>&1
echo "ba ncu rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_ba.csv $BA > gpurun_out/ncu_launches_ba.log 2>&1
echo "ba launches rc=$?"
timeout 300 $GMM > gpurun_out/bench_gmm_small.json 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_gmm.csv $GMM > gpurun_out/ncu_launches_gmm.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gmm_ -s 12 -c 6 \
    -o gpurun_out/prof_gmm $GMM > gpurun_out/ncu_full_gmm.log 2>&1
echo "gmm ncu rc=$?"
