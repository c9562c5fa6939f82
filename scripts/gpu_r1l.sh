TAG=r1l
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu_${TAG}.log 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/pytest_gpu_${TAG}.log
for v in base m3 p2 p2m3; do SKYCELL_K1=$v timeout 300 python bench.py --config c2 --steps 10 --no-cpu > gpurun_out/bench_c2_${v}_${TAG}.json 2>&1; echo "c2 $v rc=$?"; done
for c in c5d4 c5d5 c3; do timeout 300 python bench.py --config $c --steps 2 --no-cpu > gpurun_out/bench_${c}_${TAG}.json 2>&1; echo "$c rc=$?"; done
bash scripts/ncu_capture.sh prof_tree_${TAG} k_tree_query 1 -- python bench.py --config c5d4 --steps 1 --warmup 1 --no-cpu
