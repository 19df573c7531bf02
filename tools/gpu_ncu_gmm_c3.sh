#!/bin/bash
# ncu --set full (with source) of one configs[2] drop-in gradient evaluation's
# kernels (tools/gmm_one.py c3: 3 evaluations, the third captured)
mkdir -p gpurun_out
CMD="python tools/gmm_one.py c3 3"
timeout 300 $CMD > gpurun_out/gmm_one.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_gmm_" -s 12 -c 6 \
    -o gpurun_out/gmm_c3_${1:-cur} $CMD > gpurun_out/ncu_gmm_c3.log 2>&1
echo "ncu rc=$?"
