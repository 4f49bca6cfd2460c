#!/bin/bash
# Experiment builds with every source recompiled:
#   tools/build_variant_all.sh NAME "-DFLAG ..." -> lib/libfhe_NAME.so
# (for flags read by several files, e.g. the NTT pass plan).  Variant
# libraries are scratch: delete them after the experiment.
set -e
cd "$(dirname "$0")/../paper_2503_22227_b200/csrc"
NAME=$1; shift
mkdir -p build/v_$NAME
OBJS=""
for f in context ntt ntt_mm poly keyswitch behz crt philox crc32 capi; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
    --expt-relaxed-constexpr -cudart static "$@" -c $f.cu -o build/v_$NAME/$f.o &
  OBJS="$OBJS build/v_$NAME/$f.o"
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o ../lib/libfhe_$NAME.so $OBJS
echo built lib/libfhe_$NAME.so
