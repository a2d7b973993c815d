#!/bin/bash
# dev aid: build libshellular_cuda.so with -DSHL_BRICK_TRACE into tracelib/ (per-CTA phase timestamps)
set -e
cd "$(dirname "$0")/../paper_2511_04025_b200/csrc"
O=../../build/obj
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -DSHL_BRICK_TRACE -c brick.cu -o /tmp/brick_trace.o
mkdir -p ../../tracelib
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o ../../tracelib/libshellular_cuda.so $O/field.o $O/voxel.o $O/solver.o /tmp/brick_trace.o $O/shl_api.o $O/slab.o $O/geom.o $O/host_design.o -lcudart_static -lpthread -ldl -lrt
