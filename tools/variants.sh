#!/bin/bash
# Build tuning variants of libseqcdc.so into /tmp/v_<name>.so (run on the GPU box or here).
set -e
cd "$(dirname "$0")/.."
build() { name=$1; shift; nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --extended-lambda \
  -Xcompiler -fPIC -Xcompiler -fvisibility=hidden -shared "$@" -o /tmp/v_$name.so paper_2505_21194_b200/csrc/seqcdc.cu; }
for spec in "$@"; do
  name=${spec%%:*}; flags=${spec#*:}
  build $name $flags &
done
wait
