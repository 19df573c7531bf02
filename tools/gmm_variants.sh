#!/bin/bash
# GMM build variants (tools/build_variants.sh gmm.cu ...): drop-in step time at configs[2] and a d=128 shape
for lib in tools/variants/*.so; do
  echo "$(basename $lib .so): $(REVGPU_LIB=$PWD/$lib timeout 200 python tools/gmm_restore_probe.py 2>&1 | sed 's/E=.*//' | tr '\n' ' ')"
done
