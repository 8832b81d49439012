#!/bin/bash
# A/B of a kernel compile knob on the GPU box: time C3/C5 walks with the
# default build, rebuild libfrwgpu.so with FRW_NVCC_EXTRA="$1", time again.
# usage: tools/ab_build.sh "-DFRW_KMW_MINB=2" [configs...]
trap 'python -c "from paper_2507_09730_b200 import build as b; b.build_gpu_lib()" > /dev/null 2>&1' EXIT  # back to the default build
set -e
flags="$1"; shift
cfg="${@:-c3 c5}"
echo "== default"; python tools/quick_walks.py $cfg 2>&1 | grep -v "walks=100000 "
FRW_NVCC_EXTRA="$flags" python -c "from paper_2507_09730_b200 import build as b; b.build_gpu_lib(force=True)" 2>&1 | grep -E "registers" | head -40 > gpurun_out/ab_regs.txt || true
echo "== $flags"; python tools/quick_walks.py $cfg 2>&1 | grep -v "walks=100000 "
