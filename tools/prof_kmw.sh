#!/bin/bash
# ncu --set full of the first (largest) k_mw launch of the warm C3 run in
# tools/profile_walks.py.  Usage: tools/prof_kmw.sh <config> <out-name> [kernel-regex]
cfg=${1:-c3}; out=${2:-prof_kmw}; kre=${3:-k_mw}
FRW_TRACE_ROUNDS=1 python tools/profile_walks.py $cfg > gpurun_out/${out}_trace.log 2>&1 || exit 1
# k_mw launches of the first (cold) extract = its wavefront rounds
n1=$(awk '/^round 0:/{n++} n==1' gpurun_out/${out}_trace.log | grep -c " mw [0-9.]* ms$")
ncu --set full --import-source on --clock-control none -k regex:"$kre" --launch-skip $n1 --launch-count 1 \
    -o gpurun_out/$out python tools/profile_walks.py $cfg > gpurun_out/${out}_ncu.log 2>&1
echo "skip=$n1 rc=$?"
