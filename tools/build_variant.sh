#!/bin/bash
# Build a variant of libwd_b200.so with extra nvcc defines for the fast
# stage kernel (A/B timing through WD_B200_LIB):
#   tools/build_variant.sh <name> -DWD_S3_D=3 -DWD_S3_PF=2
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
CS=$ROOT/paper_2111_09859_b200/csrc
OUT=$ROOT/paper_2111_09859_b200/variants
mkdir -p "$OUT"
name=$1; shift
make -C "$CS" -j4 wd_capi.o wd_fused.o >/dev/null
nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -fmad=false \
  -Xcompiler -fPIC,-O2 -Xptxas -v --expt-relaxed-constexpr "$@" -c "$CS/wd_stage_fast.cu" \
  -o "$OUT/$name.o" 2> "$OUT/$name.ptxas.log"
nvcc -gencode arch=compute_100a,code=sm_100a -shared --cudart=static -o "$OUT/libwd_$name.so" \
  "$CS/wd_capi.o" "$CS/wd_fused.o" "$OUT/$name.o"
grep -A2 "k_f3_fast3ILi3ELb0ELi2" "$OUT/$name.ptxas.log" | grep -E "registers|spill" | tr '\n' ' '; echo
