#!/bin/bash
# Time each built variant (tools/build_variant.sh) on BASELINE configs
# through tools/bench_configs.py:  tools/ab_configs.sh c5,c3 [steps]
CASES=${1:-c5}
STEPS=${2:-5}
for so in paper_2111_09859_b200/variants/libwd_*.so; do
  n=$(basename $so .so)
  WD_B200_LIB=$PWD/$so timeout 600 python tools/bench_configs.py --cases $CASES --steps $STEPS 2>&1 | \
    python -c "
import json,sys
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: continue
    if 'ms_per_step' in d: print('$n', d['case'], d['ms_per_step'], d['state'])"
done
