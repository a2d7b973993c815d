#!/bin/bash
# dev aid: build a variant libshellular_cuda.so for same-box A/B runs
# (SHL_LIB=varlib/<name>/libshellular_cuda.so python bench.py ...).
#   tools/variant.sh <name> [command run inside a scratch copy of csrc/, e.g. a sed]
set -e
R="$(cd "$(dirname "$0")/.." && pwd)"
N=$1; shift
T=/tmp/shl_variant_$N
rm -rf $T; mkdir -p $T/paper_2511_04025_b200 $R/varlib/$N
cp -r $R/include $T/include
cp -r $R/paper_2511_04025_b200/csrc $T/paper_2511_04025_b200/csrc
if [ $# -gt 0 ]; then (cd $T/paper_2511_04025_b200/csrc && bash -c "$*"); fi
make -s -j8 -C $T/paper_2511_04025_b200/csrc OUT=$R/varlib/$N/libshellular_cuda.so OBJDIR=$T/obj
echo built $R/varlib/$N/libshellular_cuda.so
