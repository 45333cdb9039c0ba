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
# which translation unit the defines apply to: TU=wd_stage_fast (default), wd_fused, wd_capi
TU=${TU:-wd_stage_fast}
make -C "$CS" -j4 wd_capi.o wd_fused.o wd_stage_fast.o >/dev/null
FL="-O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -fmad=false -Xcompiler -fPIC,-O2 -Xptxas -v --expt-relaxed-constexpr"
nvcc $FL "$@" -c "$CS/$TU.cu" -o "$OUT/$name.o" 2> "$OUT/$name.ptxas.log"
OBJS="$OUT/$name.o"
for u in wd_capi wd_fused wd_stage_fast; do [ "$u" = "$TU" ] || OBJS="$OBJS $CS/$u.o"; done
nvcc -gencode arch=compute_100a,code=sm_100a -shared --cudart=static -o "$OUT/libwd_$name.so" $OBJS
grep -E "registers|spill" "$OUT/$name.ptxas.log" | sort | uniq -c | sort -rn | head -3
