#!/bin/bash
# Build tuning variants of libseqcdc.so into build/v_<name>.so (here or on the GPU box):
#   tools/variants.sh "name:-DFLAG=1 -DOTHER=2" ...
# Select one at run time with SEQCDC_LIB=build/v_<name>.so (tuning only).
set -e
cd "$(dirname "$0")/.."
mkdir -p build
b() { name=$1; shift; nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --extended-lambda \
  -Xcompiler -fPIC -Xcompiler -fvisibility=hidden -shared "$@" -o build/v_$name.so \
  paper_2505_21194_b200/csrc/seqcdc.cu paper_2505_21194_b200/csrc/seqcdc_range.cu paper_2505_21194_b200/csrc/seqcdc_dedup.cu; }
for spec in "$@"; do
  name=${spec%%:*}; flags=${spec#*:}
  b $name $flags &
done
wait
