#!/bin/bash
# Interpreter experiments: the full library with kernels_program.cu rebuilt under
# extra -D flags, into variants/<name>/libmcb.so (select with MCB_LIB=...).
#   tools/build_prog_variants.sh name "-DFLAG=1 ..." [name "-D..."] ...
set -e
cd "$(dirname "$0")/../paper_2104_10073_b200/csrc"
make -s -j8 >/dev/null
NV="nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -fmad=false -std=c++17 -Xcompiler -fPIC,-fvisibility=hidden -I../../include -I."
OBJS=$(ls _obj/*.o | grep -v kernels_program.o)
while [ $# -ge 2 ]; do
  d=../../variants/$1; mkdir -p $d
  $NV $2 -Xptxas -v -c kernels_program.cu -o $d/kernels_program.o 2> $d/ptxas.log &
  names="$names $1"
  shift 2
done
wait
for n in $names; do
  d=../../variants/$n
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o $d/libmcb.so $OBJS $d/kernels_program.o -Xcompiler -pthread -ldl
done
