#!/bin/bash
# DRAM bytes per kernel of ONE drop-in configs[2] evaluation (L2 evicted by a
# 256 MiB read before each evaluation, no flush between its kernels):
# gpurun_out/gmm_dram_eval.csv -> tools/gmm_dram_json.py
mkdir -p gpurun_out
timeout 300 python tools/gmm_one.py c3 3 --flush > /dev/null 2>&1 && \
timeout 600 ncu --cache-control none --clock-control none --metrics dram__bytes_read.sum,dram__bytes_write.sum \
  -k regex:"k_gmm_" --csv python tools/gmm_one.py c3 3 --flush > gpurun_out/gmm_dram_eval.csv 2>/dev/null
echo "ncu rc=$?"
