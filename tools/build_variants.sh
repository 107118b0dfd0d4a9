#!/bin/bash
# Builds eval.cu variants with extra -D flags into build/variants/lib_<name>.so.
# usage: tools/build_variants.sh name "-DFOO=1 -DBAR=2" [name2 "flags2" ...]
set -e
cd "$(dirname "$0")/.."
mkdir -p build/variants
OBJS=""
for s in model grid select dense update assemble prof scan consumers match abi; do OBJS="$OBJS build/obj/$s.cu.o"; done
while [ $# -ge 2 ]; do
  name=$1; flags=$2; shift 2
  nvcc -O3 -std=c++17 -lineinfo -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC,-ffp-contract=off \
    --expt-relaxed-constexpr -I include $flags \
    -c paper_2509_26222_b200/csrc/eval.cu -o build/variants/eval_$name.o
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -o build/variants/lib_$name.so $OBJS \
    build/variants/eval_$name.o -lcudart_static -lrt -lpthread -ldl
done
