TAG=r1f
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu_${TAG}.log 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/pytest_gpu_${TAG}.log
timeout 600 compute-sanitizer --tool memcheck --print-limit 20 python bench.py --config c5d5 --n 3000000 --rho 5 --steps 1 --warmup 1 --no-cpu > gpurun_out/sanitize_c5d5_${TAG}.log 2>&1; echo "sanitize rc=$?"; grep -m5 -A12 "Invalid\|ERROR" gpurun_out/sanitize_c5d5_${TAG}.log | head -40
for c in c2 c1 c4c c5d3 c5d4 c5d5; do timeout 300 python bench.py --config $c --steps 5 --no-cpu > gpurun_out/bench_${c}_${TAG}.json 2>&1; echo "$c rc=$?"; done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2_${TAG}.csv python bench.py --config c2 --steps 1 --warmup 3 --no-cpu > /dev/null 2>&1; echo "launch c2 rc=$?"
