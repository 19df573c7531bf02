#!/bin/bash
# generated-kernel tuning sweep (block, chunk multiple, min blocks) on the Bessel batch
for cfg in "256 8 3" "128 16 8" "128 16 6" "128 16 8" "128 16 7" "128 8 8"; do
  set -- $cfg
  echo "block=$1 M=$2 minb=$3: $(REVGPU_CODEGEN_BLOCK=$1 REVGPU_CODEGEN_M=$2 REVGPU_CODEGEN_MINB=$3 timeout 200 python tools/codegen_speed.py 26 | cut -c1-80)"
done
