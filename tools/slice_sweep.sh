#!/bin/bash
# Walk-engine round time slices and tail threshold sweep (device walks/s of
# warm 1e6-walk calls): tools/slice_sweep.sh "<mw> <adv> <tail>" ...
for cfg in "$@"; do
  set -- $cfg
  for c in ${CFGS:-c3 c5}; do
    r=$(FRW_MW_SLICE=$1 FRW_ADV_SLICE=$2 FRW_TAIL_WALKS=$3 python tools/quick_walks.py $c 2>&1 | tail -1 | grep -o "walks/s(dev)=[0-9.e+]*")
    echo "mw=$1 adv=$2 tail=$3 $c $r"
  done
done
