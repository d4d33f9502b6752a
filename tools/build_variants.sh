#!/bin/bash
# Experimental builds of libgqsa.so (W4, G = 16, B <= 2 kernels only) with
# compile-time knobs, into paper_2412_17560_b200/lib/var/<name>.so.
#   tools/build_variants.sh name "-DGQSA_BUFS=4 -DGQSA_WARPS_SMALL=12" [name2 "flags2" ...]
set -e
SRC=paper_2412_17560_b200/csrc
OUT=paper_2412_17560_b200/lib/var
mkdir -p $OUT
while [ $# -ge 2 ]; do
  name=$1; flags=$2; shift 2
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O3 \
    --expt-relaxed-constexpr -DGQSA_FAST_BUILD $flags -Xptxas -v -shared -o $OUT/$name.so \
    $SRC/gqsa_stream.cu $SRC/gqsa_tc.cu $SRC/gqsa_capi.cu $SRC/gqsa_pack.cpp $SRC/gqsa_pack_tc.cpp $SRC/gqsa_compress.cpp 2> $OUT/$name.ptxas &
done
wait
grep -h "Used" $OUT/*.ptxas | head -40
