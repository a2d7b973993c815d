#!/bin/bash
# dev aid: build libshellular_cuda.so with an alternative brick.cu (+ -D flags)
# into varlib/<name>/ for same-box A/B runs (SHL_LIB=varlib/<name>/libshellular_cuda.so)
#   tools/variant.sh <name> <brick.cu path> [-DFOO=1 ...]
set -e
R="$(cd "$(dirname "$0")/.." && pwd)"
N=$1; SRC=$2; shift 2
O=$R/build/obj; V=$R/varlib/$N
mkdir -p $V
cp "$SRC" $R/paper_2511_04025_b200/csrc/.variant_brick.cu
(cd $R/paper_2511_04025_b200/csrc && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
   -Xcompiler -ffp-contract=off --expt-relaxed-constexpr "$@" -c .variant_brick.cu -o $V/brick.o)
rm -f $R/paper_2511_04025_b200/csrc/.variant_brick.cu
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $V/libshellular_cuda.so $O/field.o $O/voxel.o $O/solver.o $V/brick.o \
   $O/shl_api.o $O/slab.o $O/geom.o $O/host_design.o -lcudart_static -lpthread -ldl -lrt
echo built $V/libshellular_cuda.so
