#!/bin/bash
# Experiment builds: tools/build_variant.sh NAME "-DFLAG ..." -> lib/libfhe_NAME.so
# (ntt.cu recompiled with the flags, linked with the default objects).
set -e
cd "$(dirname "$0")/../paper_2503_22227_b200/csrc"
make -s >/dev/null
NAME=$1; shift
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
  --expt-relaxed-constexpr -cudart static -Xptxas -v $* -c ntt.cu -o build/ntt_$NAME.o \
  2> build/ntt_$NAME.ptxas.log
nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o ../lib/libfhe_$NAME.so \
  build/context.o build/ntt_$NAME.o build/ntt_mm.o build/poly.o build/keyswitch.o build/behz.o build/capi.o
echo built lib/libfhe_$NAME.so
