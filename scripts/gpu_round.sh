# Full GPU check of a round: smoke, parity tests, bench lines for every
# BASELINE config, one launch list and one ncu --set full capture of K1
# (summarised on the box; see scripts/ncu_capture.sh).
# usage: bash scripts/gpu_round.sh <tag> [configs...]
TAG=${1:-r1}; shift
CFGS=${@:-c1 c2 c3 c4c c4i c5d2 c5d3 c5d4 c5d5 c5d6 c5d7 c5d8}
mkdir -p gpurun_out
{ nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv; nproc; lscpu | grep -E "Model name|Socket|Core"; } > gpurun_out/host_${TAG}.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_${TAG}.log 2>&1; echo "smoke rc=$?"
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu_${TAG}.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu_${TAG}.log
timeout 900 python bench.py > gpurun_out/bench_default_${TAG}.json 2> gpurun_out/bench_default_${TAG}.err; echo "bench (default) rc=$?"
timeout 900 python bench.py --impl reference > gpurun_out/bench_reference_${TAG}.json 2>&1; echo "bench reference rc=$?"
for c in $CFGS; do timeout 600 python bench.py --config $c --steps 3 --no-cpu > gpurun_out/bench_${c}_${TAG}.json 2>&1; echo "$c rc=$?"; done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2_${TAG}.csv python bench.py --steps 1 --warmup 3 --no-cpu > /dev/null 2>&1; echo "launch list rc=$?"
bash scripts/ncu_capture.sh prof_k1_c2_${TAG} k_stream 3 -- python bench.py --steps 1 --warmup 3 --no-cpu
