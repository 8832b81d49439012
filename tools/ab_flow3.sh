#!/bin/bash
# k_flow (SM roles): advance share x run-to-completion threshold
export FRW_TAIL_KERNEL=flow
for v in $1; do
  tools/use_variant.sh $v
  for tw in $2; do
    echo "== $v FRW_TAIL_WALKS=$tw"
    FRW_TAIL_WALKS=$tw python tools/quick_walks.py c3 c4 c5 2>&1 | grep "misses=0 "
  done
done
tools/use_variant.sh default
