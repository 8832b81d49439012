#!/bin/bash
# C2 headline kernel variants: device transitions/s of the bench's C2 step
# (1e7 Philox transits, L2 flushed) for FRW_GRID_WPT=1/2 and thread counts.
for t in ${T2:-768 896}; do
  FRW_NVCC_EXTRA="-DFRW_GRID_T2=$t" python -c "from paper_2507_09730_b200 import build as b; b.build_gpu_lib()" > gpurun_out/c2ab_build_$t.log 2>&1
  grep -A2 "Function properties for .*mw_grid_fast2" gpurun_out/c2ab_build_$t.log | grep -E "spill|Used" | tr '\n' ' '; echo
  for w in 1 2; do
    r=$(FRW_GRID_WPT=$w python bench.py --headline-only --no-cpu-baseline --steps 10 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('%.4e' % d['value'], '%.3f' % d['roofline']['frac'])")
    echo "T2=$t WPT=$w $r"
  done
done
python -c "from paper_2507_09730_b200 import build as b; b.build_gpu_lib()" > /dev/null 2>&1
