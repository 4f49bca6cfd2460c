#!/bin/bash
# Experiment builds: tools/build_variant.sh NAME SRC "-DFLAG ..." -> lib/libfhe_NAME.so
# (SRC, e.g. ntt or keyswitch, recompiled with the flags and linked with the
# default objects of every other file).  Variant libraries are scratch: delete
# them after the experiment (they travel to the GPU box with the snapshot).
set -e
cd "$(dirname "$0")/../paper_2503_22227_b200/csrc"
make -s >/dev/null
NAME=$1; SRC=$2; shift 2
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
  --expt-relaxed-constexpr -cudart static -Xptxas -v "$@" -c $SRC.cu -o build/${SRC}_$NAME.o \
  2> build/${SRC}_$NAME.ptxas.log
OBJS=""
for f in context ntt ntt_mm poly keyswitch behz crt philox crc32 capi; do
  if [ "$f" = "$SRC" ]; then OBJS="$OBJS build/${SRC}_$NAME.o"; else OBJS="$OBJS build/$f.o"; fi
done
nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o ../lib/libfhe_$NAME.so $OBJS
echo built lib/libfhe_$NAME.so
