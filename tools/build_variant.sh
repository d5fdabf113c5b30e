#!/bin/bash
# Build a tuning variant of the product library: tools/build_variant.sh NAME "-DFLAG=.. ..."
# -> tools/variants/NAME.so (load with P2G_LIB_PATH=tools/variants/NAME.so)
set -e
HERE=$(cd "$(dirname "$0")/.." && pwd)
C=$HERE/paper_2207_02543_b200/csrc
mkdir -p $HERE/tools/variants
/usr/local/cuda/bin/nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC \
  -ccbin /usr/bin/g++ --expt-relaxed-constexpr -Xcompiler -ffp-contract=off $2 -shared \
  -o $HERE/tools/variants/$1.so $C/p2g_solver.cu $C/p2g_pattern.cpp $C/p2g_mesh.cpp $C/p2g_partition.cpp \
  -cudart static -lpthread -Xptxas -v 2> $HERE/tools/variants/$1.ptxas.log
grep -A2 "_blk" $HERE/tools/variants/$1.ptxas.log | grep -B1 -A1 "Li2E" | grep -E "spill" | head -8 || true
