#!/bin/bash
# default build (k_flow, SM roles, measured advance share): chosen share, then a sweep of
# FRW_FLOW_ADV_PCT to check the heuristic
for c in c3 c4 c5; do
  FRW_TRACE_ROUNDS=1 timeout 120 python tools/quick_walks.py $c 2>&1 | grep "k_flow:" | tail -1 | sed "s/^/$c auto /"
done
echo "== auto"; timeout 300 python tools/quick_walks.py c3 c4 c5 2>&1 | grep "misses=0 "
for pct in 30 40 50; do
  echo "== FRW_FLOW_ADV_PCT=$pct"
  FRW_FLOW_ADV_PCT=$pct timeout 300 python tools/quick_walks.py c3 c4 c5 2>&1 | grep "misses=0 "
done
echo "== k_tail"; FRW_TAIL_KERNEL=tail FRW_TAIL_WALKS=151552 timeout 300 python tools/quick_walks.py c3 c4 c5 2>&1 | grep "misses=0 "
echo "== MWE auto"; FRW_MODE=HYBRID-MWE timeout 300 python tools/quick_walks.py c3 c5 2>&1 | grep "misses=0 "
echo "== MWE k_tail"; FRW_MODE=HYBRID-MWE FRW_TAIL_KERNEL=tail FRW_TAIL_WALKS=151552 timeout 300 python tools/quick_walks.py c3 c5 2>&1 | grep "misses=0 "
