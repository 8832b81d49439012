#!/bin/bash
# DRAM bytes of every walk-engine launch of one warm 1e6-walk call (ncu
# metrics pass, all launches; cuProfilerStart/Stop bracket the warm call)
# usage: tools/ncu_walks.sh <config> <out.csv>
cfg=${1:-c3}; out=${2:-gpurun_out/ncu_walks_$cfg.csv}
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__thread_inst_executed_per_inst_executed.ratio \
    --clock-control none --profile-from-start off --csv --log-file $out \
    python tools/profile_walks.py $cfg 1000000 > ${out%.csv}.log 2>&1
echo "$cfg rc=$?"
