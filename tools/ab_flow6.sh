#!/bin/bash
# one-kernel flow (roles by SM pair) against the two-kernel flow (flow2)
for k in flow flow2 flow flow2; do
  echo "== FRW_TAIL_KERNEL=$k"; FRW_TAIL_KERNEL=$k timeout 300 python tools/quick_walks.py c3 c4 c5 2>&1 | grep -E "misses=0 |rror"
done
for pct in 30 40 50 60; do
  echo "== flow2 FRW_FLOW_ADV_PCT=$pct"
  FRW_TAIL_KERNEL=flow2 FRW_FLOW_ADV_PCT=$pct timeout 300 python tools/quick_walks.py c3 c4 c5 2>&1 | grep -E "misses=0 |rror"
done
echo "== MWE flow2"; FRW_TAIL_KERNEL=flow2 FRW_MODE=HYBRID-MWE timeout 300 python tools/quick_walks.py c3 c5 2>&1 | grep -E "misses=0 |rror"
