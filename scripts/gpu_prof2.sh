# usage: bash scripts/gpu_prof2.sh <tag>  -- tests, bench lines, launch lists, ncu full of K4/K5/K1
TAG=${1:-p}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu_${TAG}.log 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/pytest_gpu_${TAG}.log
for c in c2 c1 c4c c5d3; do timeout 300 python bench.py --config $c --steps 5 --no-cpu > gpurun_out/bench_${c}_${TAG}.json 2>&1; echo "$c rc=$?"; done
for c in c2 c4c; do timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${c}_${TAG}.csv python bench.py --config $c --steps 1 --warmup 3 --no-cpu > /dev/null 2>&1; echo "launch $c rc=$?"; done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_candidates -s 7 -c 1 -o gpurun_out/prof_k4_${TAG} python bench.py --steps 1 --warmup 3 --no-cpu > /dev/null 2>&1; echo "ncu k4 rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_allpairs -s 7 -c 1 -o gpurun_out/prof_k5_${TAG} python bench.py --steps 1 --warmup 3 --no-cpu > /dev/null 2>&1; echo "ncu k5 rc=$?"
