#!/bin/bash
# C2 headline kernel: bench --headline-only (1e7 Philox transits, L2 flushed) per variant
for v in $1; do
  tools/use_variant.sh $v
  for rep in 1 2; do
    r=$(python bench.py --headline-only --no-cpu-baseline --steps 10 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('%.4e' % d['value'], 'e2e %.4e' % d['e2e']['value'])")
    echo "$v $r"
  done
done
tools/use_variant.sh default
