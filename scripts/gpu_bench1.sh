set -x
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu 2>&1 | tail -5
timeout 600 python bench.py --config c1 --steps 5 --warmup 3 --no-cpu 2>&1 | tail -3
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv python bench.py --steps 1 --warmup 3 --no-cpu > gpurun_out/ncu_bench.log 2>&1
tail -3 gpurun_out/ncu_bench.log
