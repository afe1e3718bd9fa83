#!/bin/bash
# Build sweep-kernel variants of libschwarz_b200.so into variants/ (git-ignored;
# they travel to the GPU box). Usage: scripts/build_variants.sh name "-DFLAG=.." ...
cd "$(dirname "$0")/.."
mkdir -p variants
while [ $# -ge 2 ]; do
  name=$1; flags=$2; shift 2
  rm -f variants/lib_$name.so
  nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo -O3 -std=c++17 -Xcompiler -fPIC,-O3 \
    -shared $flags paper_2110_03946_b200/csrc/solver.cu paper_2110_03946_b200/csrc/generators.cpp \
    -o variants/lib_$name.so -Xptxas -v 2>&1 | grep -A3 "Compiling entry.*oras_sweep_kernelIdLi[48]ELb1" | grep -o "oras_sweep_kernelIdLi[48]\|[0-9]* bytes spill stores\|Used [0-9]* registers" | tr '\n' ' '
  [ -f variants/lib_$name.so ] && echo " <- $name" || echo " <- $name FAILED"
done
