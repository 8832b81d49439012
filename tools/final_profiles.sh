#!/bin/bash
# ncu evidence of the current build (one GPU): walk kernels on C3/C5 (--set full, one launch
# each, warm 1e6-walk call), the C2 single-cube kernel, the tail walk count for per-walk DRAM,
# and the launch list of a short bench.  Outputs under gpurun_out/ (summarised into profiles/).
tag=${1:-r02f}
mkdir -p /tmp/prof
for c in c3 c5; do
  FRW_TRACE_ROUNDS=1 python tools/profile_walks.py $c 1000000 > gpurun_out/trace_${c}_${tag}.txt 2>&1
  for k in k_tail k_mw k_advance k_compile; do
    ncu --set full --import-source on --clock-control none --profile-from-start off \
        -k regex:"$k" --launch-count 1 -o /tmp/prof/prof_${k}_${c}_${tag} \
        python tools/profile_walks.py $c 1000000 > gpurun_out/prof_${k}_${c}_${tag}.log 2>&1
    echo "$c $k rc=$?"
  done
done
ncu --set full --import-source on --clock-control none -k regex:mw_grid_fast --launch-count 1 \
    -o /tmp/prof/prof_mwgrid_c2_${tag} python tools/profile_c2.py c2 > gpurun_out/prof_mwgrid_c2_${tag}.log 2>&1
echo "c2 rc=$?"
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__thread_inst_executed_per_inst_executed.ratio \
    --clock-control none -c 800 --csv --log-file gpurun_out/${tag}_launches_bench.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --walk-steps 1 --c5-walks 2000000 \
    > gpurun_out/ncu_bench_${tag}.log 2>&1
echo "launches rc=$?"
# summaries (the .ncu-rep files stay on the box: gpurun brings back at most 64 MiB)
for c in c3 c5; do
  for k in k_tail k_mw k_advance k_compile; do
    r=/tmp/prof/prof_${k}_${c}_${tag}.ncu-rep
    python tools/ncu_summary.py $r $k "$k<PHILOX>" "${c^^} HYBRID-MW, 1e6 warm walks (tools/profile_walks.py $c)" \
        "the largest $k launch of the warm run" walk.cu > gpurun_out/sum_${k}_${c}_${tag}.json 2>/dev/null
    python tools/ncu_funcs.py $r $k > gpurun_out/funcs_${k}_${c}_${tag}.txt 2>&1
  done
done
python tools/ncu_summary.py /tmp/prof/prof_mwgrid_c2_${tag}.ncu-rep mw_grid_fast "mw_grid_fast<PHILOX>" \
    "C2 41^3 block cube, 1e7 Philox transits (tools/profile_c2.py)" "one launch" mw_grid.cu \
    > gpurun_out/sum_mwgrid_c2_${tag}.json 2>/dev/null
python tools/ncu_lines.py /tmp/prof/prof_mwgrid_c2_${tag}.ncu-rep mw_grid 30 > gpurun_out/lines_mwgrid_c2_${tag}.txt 2>&1
cp /tmp/prof/prof_k_tail_c3_${tag}.ncu-rep gpurun_out/ 2>/dev/null
