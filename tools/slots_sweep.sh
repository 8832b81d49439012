#!/bin/bash
# walks/s (device) over the resident slot pool (FRW_SLOTS; default 2^20)
for cfg in ${CFGS:-c3 c5}; do
  for sl in 262144 524288 1048576; do
    r=$(FRW_SLOTS=$sl python tools/quick_walks.py $cfg 2>&1 | tail -1 | grep -o "walks/s(dev)=[0-9.e+]*")
    echo "$cfg slots=$sl $r"
  done
done
