#!/bin/bash
# Build a variant library: tools/exp/variant.sh NAME "-DFLAG ..." -> tools/exp/NAME.so
# (SRCF.cu, default attention.cu, recompiled with the extra flags and linked
# with the other objects).
set -e
cd "$(dirname "$0")/../.."
make -s -j16 >/dev/null
NAME=$1; shift
mkdir -p build/var
SRCF=${SRCF:-attention}
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 \
  -Xcompiler -fPIC --expt-relaxed-constexpr $@ -c paper_2605_21226_b200/csrc/$SRCF.cu \
  -o build/var/${SRCF}_$NAME.o
objs=$(ls build/obj/*.o | grep -v $SRCF.cu.o)
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static \
  -o tools/exp/$NAME.so build/var/${SRCF}_$NAME.o $objs -Xcompiler -pthread
echo built tools/exp/$NAME.so
