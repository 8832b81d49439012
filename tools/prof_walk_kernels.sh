#!/bin/bash
# ncu --set full of the walk engine's kernels on a warm run of a config
# (tools/profile_walks.py brackets the warm run with cuProfilerStart/Stop):
# the round-0 k_advance and k_mw launches and the k_tail launch.
# usage: tools/prof_walk_kernels.sh <config> <tag> [walks]
cfg=${1:-c3}; tag=${2:-r02}; walks=${3:-1000000}
for k in ${KERNELS:-k_tail k_mw k_advance k_compile}; do
  ncu --set full --import-source on --clock-control none --profile-from-start off \
      -k regex:"$k" --launch-count 1 -o gpurun_out/prof_${k}_${cfg}_${tag} \
      python tools/profile_walks.py $cfg $walks > gpurun_out/prof_${k}_${cfg}_${tag}.log 2>&1
  echo "$k rc=$?"
done
