# A/B timing of env switches on one config: bash scripts/ab.sh <config> <steps> "ENV=.. ENV2=.." ...
CFG=$1; STEPS=$2; shift 2
for envs in "$@"; do
  line=$(env $envs timeout 300 python bench.py --config $CFG --steps $STEPS --warmup 3 --no-cpu 2>/dev/null | tail -1)
  python - "$envs" "$line" <<'PY'
import json, sys
envs, line = sys.argv[1], sys.argv[2]
try:
    j = json.loads(line)
except Exception:
    print(f"{envs:40s} FAILED: {line[:200]}"); sys.exit()
r = j.get("roofline") or {}
km = {k: round(v, 3) for k, v in (r.get("kernels_ms") or {}).items()}
print(f"{envs:40s} ms {j['ms_per_step']:.4f}  {km}  stages {dict((k, round(v, 3)) for k, v in (j.get('stages_ms') or {}).items())}  S={j['config'].get('skyline_size')} ex={j['config'].get('points_examined')}")
PY
done
