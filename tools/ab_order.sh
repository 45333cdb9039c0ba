for o in 012 201 210 120; do
  WD_FILTER_ORDER=$o timeout 300 python bench.py --no-cpu --no-e2e --no-exact 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$o', d['value'], d['ms_per_step'], {k: round(v,3) for k,v in d['kernel_ms'].items()})"
done
