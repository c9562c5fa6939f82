# Full GPU check: smoke, parity tests, bench lines, launch list, one ncu --set full capture.
# usage: bash scripts/gpu_round.sh <tag>
TAG=${1:-r1}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi_${TAG}.txt
nproc >> gpurun_out/smi_${TAG}.txt; lscpu | grep -E "Model name|Socket|Thread|Core" >> gpurun_out/smi_${TAG}.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_${TAG}.log 2>&1; echo "smoke rc=$?"
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu_${TAG}.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu_${TAG}.log
timeout 900 python bench.py > gpurun_out/bench_c2_${TAG}.json 2> gpurun_out/bench_c2_${TAG}.err; echo "bench rc=$?"; tail -c 3000 gpurun_out/bench_c2_${TAG}.json
for c in c1 c3 c4c c4i c5d2 c5d8; do timeout 300 python bench.py --config $c --steps 5 --no-cpu > gpurun_out/bench_${c}_${TAG}.json 2>&1; echo "$c rc=$?"; done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2_${TAG}.csv python bench.py --steps 1 --warmup 3 --no-cpu > gpurun_out/ncu_launch_${TAG}.log 2>&1; echo "ncu launch rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_stream -s 3 -c 1 -o gpurun_out/prof_kstream_${TAG} python bench.py --steps 1 --warmup 3 --no-cpu > gpurun_out/prof_kstream_${TAG}.log 2>&1; echo "ncu full rc=$?"
