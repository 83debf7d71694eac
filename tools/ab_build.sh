#!/bin/bash
# Build the current csrc into an A/B variant directory:  tools/ab_build.sh NAME [EXTRA_NVCC_FLAGS]
# (then run e.g. TEMPO_B200_LIB=$PWD/_ab/NAME/libtempo_b200.so python bench.py ...)
set -e
N=$1
D=$(cd "$(dirname "$0")/.." && pwd)
mkdir -p $D/_ab/$N
make -C $D/paper_2210_10246_b200/csrc -j8 OUT=../../_ab/$N EXTRA="${2:-}" ../../_ab/$N/libtempo_b200.so >/dev/null
echo built _ab/$N
