#!/bin/bash
# Build an A/B variant of libvdfcg.so with extra nvcc defines for one source file (tools).
#   bash tools/build_variant.sh <out.so> <source.cu> -DNAME=VALUE ...
OUT=$1; SRC=$2; shift 2
B=paper_2504_14897_b200/_build
NV=/usr/local/cuda/bin/nvcc
FL="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -O2 --expt-relaxed-constexpr"
$NV $FL "$@" -c paper_2504_14897_b200/csrc/$SRC -o /tmp/variant_${SRC%.cu}.o || exit 1
OBJS=""
for o in ctx hist index em em_d2 em_d3 em_entry pack synth mtjump metrics stream multi api; do
  if [ "$o.cu" == "$SRC" ]; then OBJS="$OBJS /tmp/variant_${SRC%.cu}.o"; else OBJS="$OBJS $B/$o.o"; fi
done
$NV -gencode arch=compute_100a,code=sm_100a -shared -o $OUT $OBJS -lcudart_static -lrt -ldl -lpthread
