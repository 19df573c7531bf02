#!/bin/bash
# per-kernel device times (ncu launch list) of each GMM build variant at configs[2]
for lib in tools/variants/*.so; do
  REVGPU_LIB=$PWD/$lib timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    -k regex:"k_gmm_(fwd|rev)" python tools/gmm_one.py c3 4 2>/dev/null | grep k_gmm | \
    awk -F'","' -v n=$(basename $lib .so) '{print n, substr($5,1,20), $NF}' | tr -d '"' | tail -4
done
