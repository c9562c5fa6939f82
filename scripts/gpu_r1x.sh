python bench.py --config c5d4 --steps 5 --no-cpu 2>&1 | tail -1 | python -c "
import json,sys; l=json.loads(sys.stdin.read()); print(l['ms_per_step'], l['stages_ms'], l['roofline']['kernel_ms'])"
SKYCELL_TRACE=1 python bench.py --config c5d4 --steps 2 --warmup 3 --no-cpu 2>&1 | grep skycell | tail -24
