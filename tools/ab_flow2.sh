#!/bin/bash
# k_flow with SM-level roles: advance share and residency variants, then the
# run-to-completion threshold for the best one.  usage: tools/ab_flow2.sh "variants" best
export FRW_TAIL_KERNEL=flow
tools/ab_variants.sh "$1" c3 c4 c5
tools/use_variant.sh $2
for tw in 100000 200000 300000 450000; do
  echo "== $2 FRW_TAIL_WALKS=$tw"
  FRW_TAIL_WALKS=$tw python tools/quick_walks.py c3 c4 c5 2>&1 | grep "misses=0 "
done
tools/use_variant.sh default
