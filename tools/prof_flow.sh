#!/bin/bash
# ncu --set full of the k_flow launch of a warm 1e6-walk call (C3, C5) and the bench launch list
tag=${1:-r02h}
mkdir -p /tmp/prof
for c in c3 c5; do
  timeout 700 ncu --set full --import-source on --clock-control none --profile-from-start off \
      -k regex:"^k_flow$" --launch-count 1 -o /tmp/prof/prof_k_flow_${c}_${tag} \
      timeout 600 python tools/profile_walks.py $c 1000000 > gpurun_out/prof_k_flow_${c}_${tag}.log 2>&1
  echo "$c k_flow rc=$?"
  r=/tmp/prof/prof_k_flow_${c}_${tag}.ncu-rep
  python tools/ncu_summary.py $r k_flow "k_flow<PHILOX>" "${c^^} HYBRID-MW, 1e6 warm walks (tools/profile_walks.py $c)" \
      "the flow launch of the warm run" walk.cu > gpurun_out/sum_k_flow_${c}_${tag}.json 2>/dev/null
  python tools/ncu_funcs.py $r k_flow > gpurun_out/funcs_k_flow_${c}_${tag}.txt 2>&1
done
