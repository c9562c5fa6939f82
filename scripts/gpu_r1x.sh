timeout 2400 python -m pytest tests -q -m gpu -x 2>&1 | tail -3
for i in 1 2; do for c in c2 c4c c4i; do
  python bench.py --config $c --steps 10 --no-cpu 2>&1 | tail -1 | python -c "
import json,sys; l=json.loads(sys.stdin.read()); print('$c', round(l['ms_per_step'],3), {k:round(v,3) for k,v in l['stages_ms'].items()})"
done; done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2_r2w.csv python bench.py --config c2 --steps 1 --warmup 3 --no-cpu > /dev/null 2>&1
python scripts/ncu_summary.py list gpurun_out/launches_c2_r2w.csv gpurun_out/launches_c2_r2w.txt | grep -E "k_sample|total"
