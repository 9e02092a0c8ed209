#!/bin/sh
# Build an A/B variant of the library with extra -D flags:
#   sh tools/build_variant.sh NAME "-DSELLB_XLD=1"
# -> paper_1307_6209_b200/libsellb200_NAME.so (use with SELLB_LIB_PATH)
set -e
NAME=$1; DEFS=$2
D=paper_1307_6209_b200/csrc
B=$D/build_$NAME
mkdir -p $B
for f in $(cd $D && ls *.cu | sed 's/\.cu$//'); do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --fmad=false \
       -Xcompiler -fPIC,-O2 -Xptxas -v $DEFS -c $D/$f.cu -o $B/$f.o 2> $B/$f.ptxas.log &
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o paper_1307_6209_b200/libsellb200_$NAME.so \
     $B/*.o -lcudart_static -Xcompiler -fPIC
echo built paper_1307_6209_b200/libsellb200_$NAME.so
