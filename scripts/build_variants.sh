#!/bin/bash
# Build A/B variants of libadt.so into paper_2004_02297_b200/variants/; select at run
# time with ADT_LIB=<path>. Each argument is NAME=NVCC_DEFINES, e.g.
#   bash scripts/build_variants.sh pb4=-DADT_PACK_MIN_BLOCKS=4 pb6=-DADT_PACK_MIN_BLOCKS=6
set -e
cd "$(dirname "$0")/.."
mkdir -p paper_2004_02297_b200/variants
for v in "$@"; do
  name=${v%%=*}; defs=${v#*=}
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O3 -shared \
    -Xcompiler -pthread -lpthread -I include ${defs//,/ } -o paper_2004_02297_b200/variants/libadt_$name.so \
    paper_2004_02297_b200/csrc/adt_kernels.cu paper_2004_02297_b200/csrc/adt_host.cpp &
done
wait
ls paper_2004_02297_b200/variants
