#!/bin/bash
# walks/s (device) of C3/C5 HYBRID-MW over the run-to-completion threshold
# (FRW_TAIL_WALKS) and tail kernel (FRW_TAIL_KERNEL); last of 3 runs each
for cfg in ${@:-c3 c5}; do
  for tk in tail flow; do
    for tw in 0 75000 150000 303104 600000; do
      r=$(FRW_TAIL_KERNEL=$tk FRW_TAIL_WALKS=$tw python tools/quick_walks.py $cfg 2>&1 | tail -1 | grep -o "walks/s(dev)=[0-9.e+]*")
      echo "$cfg tail=$tk threshold=$tw $r"
    done
  done
done
