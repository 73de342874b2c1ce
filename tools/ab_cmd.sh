#!/bin/bash
# A/B a compile-time variant with an arbitrary timing command:
#   tools/ab_cmd.sh "-DFOO=1" "python tools/prof.py mactime 32 32"
set -e
DEFS="$1"
CMD="$2"
echo "== base"; eval "$CMD"
rm -f build/hx_ops.o build/hx_ntt.o build/hx_bsgs.o build/hx_encode.o
make lib NVFLAGS="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -O2 --expt-relaxed-constexpr $DEFS" > /dev/null
echo "== $DEFS"; eval "$CMD"
