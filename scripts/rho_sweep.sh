# C5 grid-resolution sweep: anti-correlated, every rho the dense bitmaps
# cover within the reference budget (grid.cpp:38-43), 1 warm-up + 2 steps.
# usage: bash scripts/rho_sweep.sh <tag> [n]
TAG=${1:-sweep}; N=${2:-100000000}
mkdir -p gpurun_out
for d in 2 3 4 5 6 7 8; do
  for rho in $(python -c "
d=$d
print(' '.join(str(r) for r in range(1, 40) if r*d <= 36 and (r-1)*d <= 32 and r*(d-1) <= 30))"); do
    timeout 240 python bench.py --config c5d$d --rho $rho --n $N --steps 2 --warmup 3 --no-cpu > gpurun_out/sweep_d${d}_r${rho}_${TAG}.json 2>&1
    echo "d=$d rho=$rho rc=$? $(tail -1 gpurun_out/sweep_d${d}_r${rho}_${TAG}.json | python -c 'import json,sys
try:
  l=json.loads(sys.stdin.read()); print(round(l["ms_per_step"],3), "ms", l["config"]["skyline_size"])
except Exception: print("-")')"
  done
done
