TAG=${1:-r2f}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu_${TAG}.log 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/pytest_gpu_${TAG}.log
for c in c2 c1 c4c c4i c5d2 c5d3 c5d4 c5d5 c3; do timeout 300 python bench.py --config $c --steps 10 --no-cpu > gpurun_out/bench_${c}_${TAG}.json 2>&1; echo "$c rc=$?"; done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2_${TAG}.csv python bench.py --config c2 --steps 1 --warmup 3 --no-cpu > /dev/null 2>&1; echo "launch c2 rc=$?"
python scripts/ncu_summary.py list gpurun_out/launches_c2_${TAG}.csv gpurun_out/launches_c2_${TAG}.txt | head -8
