timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2_r2e.csv python bench.py --config c2 --steps 1 --warmup 3 --no-cpu > /dev/null 2>&1; echo "launch c2 rc=$?"
python scripts/ncu_summary.py list gpurun_out/launches_c2_r2e.csv gpurun_out/launches_c2_r2e.txt
for c in c1 c2 c3; do python bench.py --config $c --steps 10 --no-cpu 2>&1 | tail -1 | python -c "
import json,sys; l=json.loads(sys.stdin.read()); print('$c', l['ms_per_step'], l['stages_ms'])"; done
