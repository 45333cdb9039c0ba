#!/bin/bash
# Time each built variant (tools/build_variant.sh) with bench.py, kernel ms only.
for so in paper_2111_09859_b200/variants/libwd_*.so; do
  n=$(basename $so .so)
  WD_B200_LIB=$PWD/$so timeout 300 python bench.py --no-cpu --no-e2e --no-exact "$@" 2>&1 | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$n', d['value'], d['ms_per_step'], {k: round(v,3) for k,v in d['kernel_ms'].items()})"
done
