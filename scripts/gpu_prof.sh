# usage: bash scripts/gpu_prof.sh <config> <kernel-regex> <tag>
CFG=${1:-c2}; KRE=${2:-k_stream}; TAG=${3:-r1}
timeout 600 ncu --set full --clock-control none --import-source on -k regex:$KRE -s 3 -c 1 -o gpurun_out/prof_${TAG} python bench.py --config $CFG --steps 1 --warmup 3 --no-cpu > gpurun_out/prof_${TAG}.log 2>&1
tail -2 gpurun_out/prof_${TAG}.log
