#!/bin/bash
# Bessel build variants (BJ_SPEC x BJ_MINB): parity subset + timing each.
mkdir -p gpurun_out/variants
for lib in tools/variants/*.so; do
  n=$(basename $lib .so)
  REVGPU_LIB=$PWD/$lib timeout 300 python -m pytest tests/test_bessel_gpu.py -q -x -k "golden or random or orders or edge" > gpurun_out/variants/$n.pytest.log 2>&1
  echo "$n pytest rc=$?" >> gpurun_out/variants/summary.txt
  REVGPU_LIB=$PWD/$lib timeout 300 python bench.py --no-e2e --no-cpu-baseline --steps 10 > gpurun_out/variants/$n.json 2>&1
  echo "$n $(python -c "import json;d=json.load(open('gpurun_out/variants/$n.json'));print(d['ms_per_step'], d['roofline']['frac'])")" >> gpurun_out/variants/summary.txt
done
