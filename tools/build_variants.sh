#!/bin/bash
# Builds libterralio_gpu variants of the manifold kernel launch configuration
# into build/variants/ for A/B timing (TLG_LIB_OVERRIDE=<path> selects one).
set -e
cd "$(dirname "$0")/.."
mkdir -p build/variants
OBJS=""
for s in model grid select dense update peak scan abi; do OBJS="$OBJS build/obj/$s.cu.o"; done
for v in "$@"; do
  T=${v%x*}; B=${v#*x}
  nvcc -O3 -std=c++17 -lineinfo -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC,-ffp-contract=off \
    --expt-relaxed-constexpr -I include -DTLG_MANIFOLD_THREADS=$T -DTLG_MANIFOLD_MINB=$B \
    -c paper_2509_26222_b200/csrc/eval.cu -o build/variants/eval_$v.o
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -o build/variants/lib_$v.so $OBJS \
    build/variants/eval_$v.o -lcudart_static -lrt -lpthread -ldl
done
