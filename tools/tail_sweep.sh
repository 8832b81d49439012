#!/bin/bash
# walks/s (device) of C3/C5 HYBRID-MW over the run-to-completion threshold
# (FRW_TAIL_WALKS; default sm_count*2048 = 303104 on a B200)
for cfg in ${CFGS:-c3 c5}; do
  for tw in ${TWS:-100000 150000 200000 303104 400000}; do
    r=$(FRW_TAIL_WALKS=$tw python tools/quick_walks.py $cfg 2>&1 | tail -1 | grep -o "walks/s(dev)=[0-9.e+]*")
    echo "$cfg threshold=$tw $r"
  done
done
