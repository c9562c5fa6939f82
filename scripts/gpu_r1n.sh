TAG=${1:-r2l}
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu_${TAG}.log 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/pytest_gpu_${TAG}.log
for c in c2 c4c c4i c1 c5d2 c5d3 c5d4 c5d5 c3; do timeout 300 python bench.py --config $c --steps 10 --no-cpu > gpurun_out/bench_${c}_${TAG}.json 2>&1; echo "$c rc=$?"; done
for r in 12 14 16 17; do timeout 300 python bench.py --config c5d2 --rho $r --steps 2 --no-cpu > gpurun_out/bench_c5d2_rho${r}_${TAG}.json 2>&1; echo "d2 rho $r rc=$? $(tail -1 gpurun_out/bench_c5d2_rho${r}_${TAG}.json | cut -c1-120)"; done
