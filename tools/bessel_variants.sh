#!/bin/bash
# Bessel build variants: device ms per 2^26 launch (best of the last three)
for lib in tools/variants/*.so; do
  echo "$(basename $lib .so): $(REVGPU_LIB=$PWD/$lib timeout 200 python tools/bessel_one.py 26 6 | tail -3 | sed 's/(67108864 z)//' | tr '\n' ' ')"
done
