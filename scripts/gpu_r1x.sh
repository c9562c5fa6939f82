SKYCELL_TRACE=1 python bench.py --config c3 --steps 1 --warmup 1 --no-cpu 2>&1 | grep skycell | tail -14
bash scripts/ncu_capture.sh prof_tree_c3_r2a k_tree_query 1 -- python bench.py --config c3 --steps 1 --warmup 1 --no-cpu
python -c "
import json; j=json.load(open('gpurun_out/prof_tree_c3_r2a.json')); m=j['metrics']
print({k.split('.')[0]:m[k]['value'] for k in m})"
