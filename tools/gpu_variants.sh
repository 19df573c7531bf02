#!/bin/bash
# build variants: parity subset + timing each (workload from $VW, tests from $VT)
mkdir -p gpurun_out/variants; : > gpurun_out/variants/summary.txt
for lib in tools/variants/*.so; do
  n=$(basename $lib .so)
  REVGPU_LIB=$PWD/$lib timeout 300 python -m pytest $VT -q -x > gpurun_out/variants/$n.pytest.log 2>&1
  echo "$n pytest rc=$?" >> gpurun_out/variants/summary.txt
  REVGPU_LIB=$PWD/$lib timeout 300 python bench.py --workload $VW --no-e2e --no-cpu-baseline --steps 20 > gpurun_out/variants/$n.json 2>&1
  echo "$n $(python -c "import json;d=json.load(open('gpurun_out/variants/$n.json'));print(d['ms_per_step'], d['roofline']['frac'])")" >> gpurun_out/variants/summary.txt
done
