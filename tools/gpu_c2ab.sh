# C2 A/B of prebuilt variants (tools/build_variant.py), then the single-cube
# parity suites under the first variant named in $2
V=${1:-"default pb2"}; T=${2:-pb2}
tools/c2_variants.sh "$V" > gpurun_out/c2ab.txt 2>&1
tools/use_variant.sh $T
python -m pytest -q -m gpu -p no:cacheprovider tests/test_gpu_microwalk.py tests/test_gpu_transit_api.py > gpurun_out/c2ab_tests.log 2>&1
tail -2 gpurun_out/c2ab_tests.log
tools/use_variant.sh default
cat gpurun_out/c2ab.txt
