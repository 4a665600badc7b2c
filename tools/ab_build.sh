#!/bin/bash
# A/B helper: tools/ab_build.sh NAME [-DFLAG ...] -> ab/libNAME.so (kernels.cu and
# context.cu rebuilt with the flags, other objects from build/obj). Dev tool only.
set -e
cd "$(dirname "$0")/.."
name=$1; shift
mkdir -p ab build/ab
for src in kernels context; do
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Iinclude \
  -Ipaper_2203_00459_b200/csrc "$@" -c paper_2203_00459_b200/csrc/$src.cu -o build/ab/${src}_$name.o &
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o ab/lib$name.so build/ab/kernels_$name.o build/ab/context_$name.o \
  $(ls build/obj/*.o | grep -v -E '/(kernels|context).o$') -lcudart
