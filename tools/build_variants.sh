#!/bin/bash
# Build librevgpu.so variants with different besselj.cu / ba.cu macros into
# tools/variants/<name>.so (for tools/gpu_variants.sh).
# usage: tools/build_variants.sh file.cu name1 "-DFOO=1" name2 "-DFOO=2" ...
set -e
cd "$(dirname "$0")/../paper_2003_04617_b200/csrc"
make -s >/dev/null
src=$1; shift
stem=$(basename $src .cu)
mkdir -p ../../tools/variants build/var
rm -f ../../tools/variants/*.so
FM=""; case $stem in besselj|ba) FM=-fmad=false;; esac
while [ $# -gt 0 ]; do
  name=$1; defs=$2; shift 2
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 \
    -Xcompiler -fPIC,-O2 -Xptxas -v $FM $defs -c $src -o build/var/$stem.$name.o 2> build/var/$name.ptxas.txt
  objs=""
  for o in capi besselj ba gmm; do
    if [ $o = $stem ]; then objs="$objs build/var/$stem.$name.o"; else objs="$objs build/$o.o"; fi
  done
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static \
    -o ../../tools/variants/$name.so $objs
  echo "$name: $(grep -A1 "k_besselj\|k_ba_jac" build/var/$name.ptxas.txt | grep -o 'Used [0-9]* registers\|[0-9]* bytes spill stores' | tr '\n' ' ')"
done
