TAG=r1g
mkdir -p gpurun_out
for c in c2 c1 c4c c5d3 c5d4; do timeout 300 python bench.py --config $c --steps 5 --no-cpu > gpurun_out/bench_${c}_${TAG}.json 2>&1; echo "$c rc=$?"; done
for c in c2 c5d4 c1; do SKYCELL_TRACE=1 timeout 300 python bench.py --config $c --steps 1 --warmup 3 --no-cpu 2>&1 | grep skycell | tail -14 > gpurun_out/trace_${c}_${TAG}.txt; echo "== trace $c"; cat gpurun_out/trace_${c}_${TAG}.txt; done
SKYCELL_K5=lists timeout 200 python bench.py --config c5d5 --steps 1 --warmup 1 --no-cpu > gpurun_out/bench_c5d5_lists_${TAG}.json 2>&1; echo "c5d5 lists rc=$?"; tail -2 gpurun_out/bench_c5d5_lists_${TAG}.json | cut -c1-400
SKYCELL_TRACE=1 SKYCELL_K5=tree timeout 300 python bench.py --config c5d5 --steps 1 --warmup 1 --no-cpu > gpurun_out/bench_c5d5_tree_${TAG}.json 2>&1; echo "c5d5 tree rc=$?"; grep skycell gpurun_out/bench_c5d5_tree_${TAG}.json | tail -20; tail -2 gpurun_out/bench_c5d5_tree_${TAG}.json | cut -c1-400
SKYCELL_K5=tree timeout 900 compute-sanitizer --tool memcheck --print-limit 10 python bench.py --config c5d5 --n 30000000 --rho 5 --steps 1 --warmup 1 --no-cpu > gpurun_out/sanitize2_${TAG}.log 2>&1; echo "sanitize rc=$?"; grep -m3 -A15 "Invalid" gpurun_out/sanitize2_${TAG}.log | head -50; tail -3 gpurun_out/sanitize2_${TAG}.log
