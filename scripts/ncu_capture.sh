# usage: bash scripts/ncu_capture.sh <name> <kernel-regex> <skip> -- <command...>
# One ncu --set full capture, summarised ON THE BOX (the .ncu-rep is ~30 MB and
# gpurun only copies back 64 MiB): writes gpurun_out/<name>.json (key metrics)
# and gpurun_out/<name>_src.csv.gz (per-SASS-line counters), removes the rep.
NAME=$1; KRE=$2; SKIP=$3; shift 4
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$KRE -s $SKIP -c 1 -o gpurun_out/$NAME "$@" > gpurun_out/$NAME.log 2>&1
echo "ncu $NAME rc=$?"
python scripts/ncu_summary.py rep gpurun_out/$NAME.ncu-rep gpurun_out/$NAME.json > /dev/null 2>&1
ncu -i gpurun_out/$NAME.ncu-rep --page source --csv --print-source sass 2>/dev/null | gzip > gpurun_out/${NAME}_src.csv.gz
rm -f gpurun_out/$NAME.ncu-rep
