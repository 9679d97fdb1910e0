#!/bin/bash
# A/B build of prefill.cu with extra flags into abtest/NAME (select it with MKV_LIB_PATH)
set -e
cd "$(dirname "$0")/.."
name=$1; shift
out=abtest/$name; mkdir -p $out
ARCH="-gencode arch=compute_100a,code=sm_100a"
FL="$ARCH -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O3 -Iinclude -Xptxas -warn-spills"
nvcc $FL "$@" -c -o $out/prefill.o paper_2411_18077_b200/csrc/prefill.cu
objs="$out/prefill.o"
for o in paper_2411_18077_b200/build/*.o; do case $(basename $o) in prefill.o) ;; *) objs="$objs $o";; esac; done
nvcc $ARCH -shared -o $out/libminikv_b200.so $objs
echo built $out
