#!/bin/bash
# A/B helper: tools/ab_build.sh NAME [-DFLAG ...] -> ab/libNAME.so (kernels.cu
# rebuilt with the flags, other objects from build/obj). Dev tool only.
set -e
cd "$(dirname "$0")/.."
name=$1; shift
mkdir -p ab build/ab
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Iinclude \
  -Ipaper_2203_00459_b200/csrc "$@" -c paper_2203_00459_b200/csrc/kernels.cu -o build/ab/k_$name.o
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o ab/lib$name.so build/ab/k_$name.o \
  build/obj/context.o build/obj/synth.o build/obj/dropin.o build/obj/fscn_io.o build/obj/generic_n.o -lcudart
