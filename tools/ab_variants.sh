#!/bin/bash
# A/B of prebuilt variants (tools/build_variant.py): device walks/s of warm
# 1e6-walk calls on the given configs.  usage: tools/ab_variants.sh "v1 v2 ..." [configs]
vars=$1; shift
cfg=${@:-c3 c4 c5}
tools/use_variant.sh default
for v in $vars; do
  tools/use_variant.sh $v
  for rep in 1 2; do
    echo "== $v (rep $rep)"; python tools/quick_walks.py $cfg 2>&1 | grep -v "walks=100000 " | sed 's/ stats=.*steps/ steps/'
  done
done
tools/use_variant.sh default
