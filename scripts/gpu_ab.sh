# usage: bash scripts/gpu_ab.sh <tag>  -- tests (tree K5), A/B bench lists vs tree, launch list
TAG=${1:-ab}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu_${TAG}.log 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/pytest_gpu_${TAG}.log
for mode in tree lists; do for c in c2 c1 c4c c5d3; do SKYCELL_K5=$mode timeout 300 python bench.py --config $c --steps 5 --no-cpu > gpurun_out/bench_${c}_${mode}_${TAG}.json 2>&1; echo "$mode $c rc=$?"; done; done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2_${TAG}.csv python bench.py --config c2 --steps 1 --warmup 3 --no-cpu > /dev/null 2>&1; echo "launch c2 rc=$?"
for c in c5d4 c5d5 c3; do timeout 240 python bench.py --config $c --steps 3 --warmup 3 --no-cpu > gpurun_out/bench_${c}_tree_${TAG}.json 2>&1; echo "tree $c rc=$?"; done
