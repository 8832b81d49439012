#!/bin/bash
# Times C3/C5 walks for several compile variants of libfrwgpu.so on the GPU
# box: tools/ab_multi.sh "<flags1>" "<flags2>" ...  ("" = default build)
trap 'python -c "from paper_2507_09730_b200 import build as b; b.build_gpu_lib()" > /dev/null 2>&1' EXIT  # back to the default build
for flags in "$@"; do
  FRW_NVCC_EXTRA="$flags" python -c "from paper_2507_09730_b200 import build as b; b.build_gpu_lib(force=True)" > /dev/null 2>&1
  for cfg in ${CFGS:-c3 c5}; do
    r=$(python tools/quick_walks.py $cfg 2>&1 | tail -1 | grep -o "walks/s(dev)=[0-9.e+]*")
    echo "[$flags] $cfg $r"
  done
done
