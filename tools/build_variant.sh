#!/bin/bash
# Build a tuning variant of libdawn.so with extra -D flags, for A/B timing via DAWN_LIB:
#   bash tools/build_variant.sh NAME "-DDAWN_BATCH_U=2 ..."   -> paper_2306_07872_b200/libdawn_NAME.so
set -e
cd "$(dirname "$0")/.."
name=$1; shift
flags="$*"
out=paper_2306_07872_b200/_build/var_$name
mkdir -p $out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC $flags -c \
  -o $out/dawn.o paper_2306_07872_b200/csrc/dawn.cu
g++ -O2 -std=c++17 -fPIC -c -o $out/oracles.o paper_2306_07872_b200/csrc/dawn_host_oracles.cpp
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o paper_2306_07872_b200/libdawn_$name.so $out/dawn.o $out/oracles.o -lcudart
echo built paper_2306_07872_b200/libdawn_$name.so
