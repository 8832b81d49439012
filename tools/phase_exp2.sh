#!/bin/bash
for c in c3 c5; do
  tools/use_variant.sh phase
  echo "=== $c normal (rounds + tail)"; python tools/profile_walks.py $c 1000000 2>&1 | tail -17
  tools/use_variant.sh phasesolo
  echo "=== $c solo lanes (one walk per warp), all in k_tail, 1e5 walks"; FRW_TAIL_WALKS=1000000000 python tools/profile_walks.py $c 100000 2>&1 | tail -17
done
tools/use_variant.sh solo
FRW_TAIL_WALKS=1000000000 ncu --set full --import-source on --clock-control none --profile-from-start off \
  -k regex:k_tail --launch-count 1 -o gpurun_out/prof_ktail_solo_c3 python tools/profile_walks.py c3 100000 > gpurun_out/prof_ktail_solo_c3.log 2>&1
tools/use_variant.sh default
tools/prof_walk_kernels.sh c3 r02
