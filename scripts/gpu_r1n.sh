TAG=r1o
mkdir -p gpurun_out
for b in 0 1; do for c in c2 c4c c5d3 c5d4 c5d5; do SKYCELL_TESTB=$b timeout 300 python bench.py --config $c --steps 5 --no-cpu > gpurun_out/bench_${c}_b${b}_${TAG}.json 2>&1; echo "b$b $c rc=$?"; done; done
for fs in 262144 65536; do for c in c2 c4i; do SKYCELL_TESTB=0 SKYCELL_FSAMPLE=$fs timeout 300 python bench.py --config $c --steps 5 --no-cpu > gpurun_out/bench_${c}_fs${fs}_${TAG}.json 2>&1; echo "fs$fs $c rc=$?"; done; done
SKYCELL_TESTB=0 SKYCELL_K5=tree timeout 300 python bench.py --config c2 --steps 5 --no-cpu > gpurun_out/bench_c2_tree_${TAG}.json 2>&1; echo "tree c2 rc=$?"
