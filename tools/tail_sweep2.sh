#!/bin/bash
# tail threshold / slice / tail-kernel sweep of warm 1e6-walk calls (device walks/s)
for c in ${CFGS:-c3 c5}; do
  for tw in 50000 100000 150000 200000 303104 450000; do
    echo "== $c FRW_TAIL_WALKS=$tw"; FRW_TAIL_WALKS=$tw python tools/quick_walks.py $c 2>&1 | grep -v "walks=100000 " | grep "misses=0 " | sed 's/ stats=.*steps/ steps/'
  done
  for sl in "32 8" "128 32" "256 64"; do
    set -- $sl
    echo "== $c FRW_MW_SLICE=$1 FRW_ADV_SLICE=$2"; FRW_MW_SLICE=$1 FRW_ADV_SLICE=$2 python tools/quick_walks.py $c 2>&1 | grep -v "walks=100000 " | grep "misses=0 " | sed 's/ stats=.*steps/ steps/'
  done
  echo "== $c FRW_TAIL_KERNEL=flow"; FRW_TAIL_KERNEL=flow python tools/quick_walks.py $c 2>&1 | grep -v "walks=100000 " | grep "misses=0 " | sed 's/ stats=.*steps/ steps/'
done
