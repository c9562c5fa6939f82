# Round-end GPU check: smoke, the GPU tests, the driver's default bench line and
# the reference arm, one bench line per BASELINE config, the C2 launch list and
# ncu --set full summaries of K1, K4a and K5 (phase B) at C2.
# usage: bash scripts/gpu_final.sh <tag>
TAG=${1:-final}
mkdir -p gpurun_out
{ nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv; nproc; lscpu | grep -E "Model name|Socket|Core"; } > gpurun_out/host_${TAG}.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_${TAG}.log 2>&1; echo "smoke rc=$?"
timeout 1200 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu_${TAG}.txt 2>&1; echo "tests_rc=$?" >> gpurun_out/pytest_gpu_${TAG}.txt; tail -2 gpurun_out/pytest_gpu_${TAG}.txt
timeout 900 python bench.py > gpurun_out/bench_default_${TAG}.jsonl 2> gpurun_out/bench_default_${TAG}.err; echo "bench default rc=$?"
timeout 1200 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_reference_${TAG}.jsonl 2>&1; echo "bench reference rc=$?"
for c in c1 c2 c2c c3 c4ishard c4cshard c5d2 c5d3 c5d4 c5d5 c5d6 c5d7 c5d8; do timeout 600 python bench.py --config $c --steps 5 --no-cpu > gpurun_out/bench_${c}_${TAG}.jsonl 2>&1; echo "$c rc=$?"; done
timeout 600 python bench.py --config c5d8 --rho 5 --steps 2 --no-cpu > gpurun_out/bench_c5d8_rho5_${TAG}.jsonl 2>&1; echo "c5d8 rho5 rc=$?"
TIMELINE=1 GAPS=5 timeout 300 python scripts/gap_probe.py > gpurun_out/timeline_c2_${TAG}.txt 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2_${TAG}.csv python bench.py --steps 1 --warmup 3 --no-cpu > /dev/null 2>&1; echo "launch list rc=$?"
bash scripts/ncu_capture.sh ${TAG}_k1_kstream_c2 k_stream 3 -- python bench.py --steps 1 --warmup 3 --no-cpu
bash scripts/ncu_capture.sh ${TAG}_k4a_candhead_c2 k_cand_head 3 -- python bench.py --steps 1 --warmup 3 --no-cpu
bash scripts/ncu_capture.sh ${TAG}_k5_long_c2 k_allpairs_long 7 -- python bench.py --steps 1 --warmup 3 --no-cpu
