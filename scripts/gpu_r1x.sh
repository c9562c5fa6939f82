timeout 2400 python -m pytest tests -q -m gpu -x 2>&1 | tail -3
for c in c2 c4c c4i c5d3 c5d4 c1; do
  python bench.py --config $c --steps 10 --no-cpu 2>&1 | tail -1 | python -c "
import json,sys; l=json.loads(sys.stdin.read()); print('$c', round(l['ms_per_step'],3), {k:round(v,3) for k,v in l['stages_ms'].items()}, l['survivors'])"
done
