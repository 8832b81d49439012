#!/bin/bash
# phase-clock breakdown of the walk engine (variants from tools/build_variant.py)
# usage: tools/phase_exp.sh [configs]
cfgs=${@:-c3 c5}
for c in $cfgs; do
  tools/use_variant.sh phase
  echo "=== $c normal (rounds + tail)"; FRW_TRACE_ROUNDS=1 python tools/profile_walks.py $c 1000000 2>&1 | grep -v "^  resolved" | tail -40
  echo "=== $c all walks in k_tail"; FRW_TAIL_WALKS=1000000000 python tools/profile_walks.py $c 1000000 2>&1 | tail -14
  tools/use_variant.sh phasesolo
  echo "=== $c solo lanes (one walk per warp), all in k_tail, 1e5 walks"; FRW_TAIL_WALKS=1000000000 python tools/profile_walks.py $c 100000 2>&1 | tail -14
done
tools/use_variant.sh default
