timeout 2400 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "large or variants" 2>&1 | tail -2
for np in 2 4; do for c in c3 c5d5 c5d4; do
  SKYCELL_PREPASSES=$np python bench.py --config $c --steps 3 --no-cpu 2>&1 | tail -1 | python -c "
import json,sys; l=json.loads(sys.stdin.read()); print('$np $c', round(l['ms_per_step'],3), {k:round(v,3) for k,v in l['stages_ms'].items()})"
done; done
