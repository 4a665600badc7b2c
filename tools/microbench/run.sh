#!/bin/bash
# build + run the exchange micro-benchmarks on the GPU box: bash tools/microbench/run.sh > out.json
set -e
cd "$(dirname "$0")/../.."
mkdir -p build/micro
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Ipaper_2203_00459_b200/csrc -Xptxas -v \
  tools/microbench/shfl_ab.cu -o build/micro/shfl_ab 2> build/micro/shfl_ab.ptxas
./build/micro/shfl_ab
