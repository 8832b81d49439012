#!/bin/bash
# compute-sanitizer over the GPU parity tests: memcheck or
# racecheck/synccheck of every kernel the selected tests launch.
# usage: tools/sanitize.sh <tool> <out-prefix> [pytest -k expression]
tool=${1:-memcheck}; out=${2:-gpurun_out/sanitize_$tool}; sel=${3:-}
CS=/usr/local/cuda/bin/compute-sanitizer
args="--tool $tool --error-exitcode 99 --print-limit 200"
[ "$tool" = memcheck ] && args="$args --leak-check no"
# small sizes: the instrumented kernels run 10-100x slower
export FRW_SAN_SMALL=1
$CS $args --log-file $out.log python -m pytest -q -m gpu -p no:cacheprovider -x \
    ${sel:+-k "$sel"} tests/test_gpu_walks.py tests/test_gpu_microwalk.py tests/test_gpu_caps.py \
    tests/test_gpu_fdm.py tests/test_gpu_sgf_solver.py > $out.pytest.log 2>&1
rc=$?
echo "compute-sanitizer $tool rc=$rc" | tee $out.rc
grep -E "ERROR SUMMARY|RACECHECK SUMMARY|Invalid|Race|Hazard" $out.log | sort | uniq -c | head -20
tail -3 $out.pytest.log
