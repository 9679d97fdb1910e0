#!/bin/bash
# A/B builds for GPU experiments: tools/abbuild.sh NAME [nvcc flags...]
# Recompiles decode.cu and capi.cu with the extra flags and links them with the other
# objects of the main build into abtest/NAME/libminikv_b200.so (select it with MKV_LIB_PATH).
set -e
cd "$(dirname "$0")/.."
name=$1; shift
out=abtest/$name; mkdir -p $out
make -s -C paper_2411_18077_b200 >/dev/null
ARCH="-gencode arch=compute_100a,code=sm_100a"
FL="$ARCH -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O3 -Iinclude -Xptxas -warn-spills"
for s in decode capi; do nvcc $FL "$@" -c -o $out/$s.o paper_2411_18077_b200/csrc/$s.cu & done; wait
objs="$out/decode.o $out/capi.o"
for o in paper_2411_18077_b200/build/*.o; do case $(basename $o) in decode.o|capi.o) ;; *) objs="$objs $o";; esac; done
nvcc $ARCH -shared -o $out/libminikv_b200.so $objs
echo "built $out/libminikv_b200.so"
