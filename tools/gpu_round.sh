#!/bin/bash
# Round evidence on one GPU: the GPU test suite, smoke(), the default bench
# line, and the ncu launch list of a short bench run (per-launch times).
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --no-e2e \
  --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1; echo "ncu rc=$?" >> gpurun_out/ncu_bench.log
# the N>1 path (shards, all_reduce, max-over-ranks, shard e2e) functionally,
# both ranks folded onto this one GPU over gloo: timings meaningless
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
  --master-port 29511 bench.py --gpus 2 --dist-backend gloo --steps 3 --warmup 3 \
  > gpurun_out/bench_gloo2.json 2> gpurun_out/bench_gloo2.err; echo "gloo2 rc=$?" >> gpurun_out/bench_gloo2.err
tail -2 gpurun_out/pytest_gpu.log; tail -1 gpurun_out/smoke.log; tail -1 gpurun_out/bench.err; tail -1 gpurun_out/ncu_bench.log; tail -1 gpurun_out/bench_gloo2.err
