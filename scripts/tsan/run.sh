#!/bin/bash
# ThreadSanitizer stress of the host packer's worker pool (no GPU needed):
# 4 caller threads x 30 adt_pack_host calls with 1..9 threads each, sleeping
# now and then so the workers go through spin -> sleep -> wake; every result
# must equal the single-threaded one byte for byte (sums bit for bit).
#   bash scripts/tsan/run.sh   (prints "mismatches 0" twice and no TSAN report)
set -e
D=$(cd "$(dirname "$0")" && pwd); R=$(dirname "$(dirname "$D")"); O=${TMPDIR:-/tmp}/adt_tsan; mkdir -p $O
echo 'extern "C" int adt_unpack(const void *, int, const unsigned char *, void *) { return -1; }' > $O/stub.cpp
g++ -O1 -g -fsanitize=thread -std=c++17 -I$R/include -I/usr/local/cuda/include $R/paper_2004_02297_b200/csrc/adt_host.cpp \
    $D/host_stress.cpp $O/stub.cpp -o $O/host_stress -L/usr/local/cuda/lib64 -lcudart -lpthread
for s in 0 200; do ADT_HOST_SPIN_US=$s LD_LIBRARY_PATH=/usr/local/cuda/lib64 $O/host_stress; done
