#!/bin/bash
# k_tail residency A/B: resident 256-thread tail CTAs per SM (launch bounds
# cap the registers), C3/C5 device walks/s of warm 1e6-walk calls
for b in ${BLOCKS:-2 3 4}; do
  FRW_NVCC_EXTRA="-DFRW_TAIL_BLOCKS=$b" python -c "from paper_2507_09730_b200 import build as b; b.build_gpu_lib()" > gpurun_out/tailab_build_$b.log 2>&1
  regs=$(grep -A2 "Function properties for .*k_tailILi1" gpurun_out/tailab_build_$b.log | grep -E "spill|Used" | tr '\n' ' ')
  echo "blocks=$b $regs"
  for c in c3 c5; do
    python tools/jump_stats.py $c 2>&1 | tail -1 | sed "s/^/  blocks=$b /"
  done
done
python -c "from paper_2507_09730_b200 import build as b; b.build_gpu_lib()" > /dev/null 2>&1
