#!/bin/bash
# Build A/B variants of libadt.so (stages x CTAs/SM of the TMA pipeline) into
# paper_2004_02297_b200/variants/; select one at run time with ADT_LIB=<path>.
set -e
cd "$(dirname "$0")/.."
mkdir -p paper_2004_02297_b200/variants
for v in "$@"; do   # e.g. s4c2 s3c3 s2c4 s6c2
  S=${v#s}; S=${S%c*}; C=${v#*c}
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O3 -shared \
    -I include -DADT_TMA_STAGES=$S -DADT_TMA_CTAS=$C \
    -o paper_2004_02297_b200/variants/libadt_$v.so paper_2004_02297_b200/csrc/adt_kernels.cu &
done
wait
ls -la paper_2004_02297_b200/variants
