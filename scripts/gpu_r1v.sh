bash scripts/ncu_capture.sh prof_tree_r1v k_tree_query 1 -- python bench.py --config c5d4 --steps 1 --warmup 1 --no-cpu
