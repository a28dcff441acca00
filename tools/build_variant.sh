#!/bin/bash
# A/B build of libcct.so with compile-time defaults flipped:  bash tools/build_variant.sh NAME "-DMACRO=V ..."
# -> abtest/NAME/libcct.so (load it with CCT_LIB_DIR=abtest/NAME; abtest/ travels with gpurun)
set -eu
ROOT="$(cd "$(dirname "${BASH_SOURCE[0]}")/.." && pwd)"
NAME=$1; FLAGS=$2
SRC=$ROOT/paper_1504_04343_b200/csrc; OBJ=$ROOT/paper_1504_04343_b200/_lib/obj; OUT=$ROOT/abtest/$NAME
mkdir -p $OUT/obj
make -s -C $SRC -j"$(nproc)"
for f in dgrad gather; do  # the sources holding the overridable defaults
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -fvisibility=hidden \
    -I$ROOT/include -I$SRC --expt-relaxed-constexpr $FLAGS -c $SRC/$f.cu -o $OUT/obj/$f.o &
done
wait
OBJS=$(ls $OBJ/*.o | grep -v -e /dgrad.o -e /gather.o -e host_)
nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o $OUT/libcct.so $OBJS $OUT/obj/dgrad.o $OUT/obj/gather.o -lpthread -ldl -lrt
rm -rf $OUT/obj
ls -la $OUT
