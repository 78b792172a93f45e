#!/bin/bash
# Builds A/B variants of the library: tools/r03_variants.sh NAME "-DLAT_X=.. ..." [NAME2 "flags2" ...]
# Only the config-4 instantiation units (lat_inst_12 / lat_inst_13) are recompiled with the flags;
# everything else links from the in-tree build.  Output: ab/NAME.so
set -eu
cd "$(dirname "$0")/.."
C=${SRCDIR:-paper_2603_16014_b200/csrc}; O=paper_2603_16014_b200/csrc
F="-gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC -Xcompiler -fvisibility=hidden -Xptxas -v --expt-relaxed-constexpr"
mkdir -p ab /tmp/ab
while [ $# -ge 2 ]; do
  name=$1; flags=$2; shift 2
  (
    for u in 12 13; do
      nvcc $F $flags -c $C/lat_inst_$u.cu -o /tmp/ab/${name}_$u.o 2> /tmp/ab/${name}_$u.log &
    done
    wait
    others=$(ls $O/_build/*.o | grep -v -E "lat_inst_1[23]\.o")
    nvcc -gencode arch=compute_100a,code=sm_100a -shared -o ab/$name.so $others /tmp/ab/${name}_12.o /tmp/ab/${name}_13.o -lcudart
    echo "built ab/$name.so"
  ) &
done
wait
