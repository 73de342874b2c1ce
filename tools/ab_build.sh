#!/bin/bash
# A/B a compile-time kernel variant on the GPU box: time the current build,
# rebuild libhx_b200.so with extra nvcc defines, time again.
#   tools/ab_build.sh "-DHX_ROWINNER_MINB=4" [batch]
set -e
DEFS="$1"
B=${2:-256}
HX_TAG=base python tools/ks_time.py $B
rm -f build/hx_ops.o build/hx_ntt.o build/hx_bsgs.o build/hx_encode.o
make lib NVFLAGS="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -O2 --expt-relaxed-constexpr $DEFS" > /dev/null
HX_TAG="$DEFS" python tools/ks_time.py $B
