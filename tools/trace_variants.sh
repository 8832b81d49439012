#!/bin/bash
# per-round trace (FRW_TRACE_ROUNDS) of a warm 1e6-walk call for each variant
vars=$1; shift
cfg=${@:-c3}
for v in $vars; do
  tools/use_variant.sh $v
  for c in $cfg; do
    echo "== $v $c"; FRW_TRACE_ROUNDS=1 python tools/profile_walks.py $c 1000000 2>&1 | grep -v "^  resolved" | tail -16
  done
done
tools/use_variant.sh default
