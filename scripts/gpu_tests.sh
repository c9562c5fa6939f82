# usage: bash scripts/gpu_tests.sh <tag> [configs...]
TAG=${1:-t}; shift
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu_${TAG}.log 2>&1
echo "pytest rc=$?"; tail -15 gpurun_out/pytest_gpu_${TAG}.log
for c in c2 "$@"; do timeout 300 python bench.py --config $c --steps 5 --no-cpu > gpurun_out/bench_${c}_${TAG}.json 2>&1; echo "$c rc=$?"; tail -c 900 gpurun_out/bench_${c}_${TAG}.json; echo; done
