CFG=${1:-c2}
timeout 300 python bench.py --config $CFG --steps 5 --warmup 3 --no-cpu 2>&1 | tail -1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${CFG}.csv python bench.py --config $CFG --steps 1 --warmup 3 --no-cpu > /dev/null 2>&1
