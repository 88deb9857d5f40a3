#!/bin/bash
# usage: scripts/ab_env.sh WORKLOAD "ENV=.. ENV2=.." ["ENV=.."...]  -> one summary line per env set
w=$1; shift
mkdir -p gpurun_out
for envs in "$@"; do
  tag=$(echo "$w $envs" | tr ' =/' '___')
  env $envs timeout 300 python bench.py --workload $w --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/ab_$tag.log 2>&1
  python - "$w" "$envs" "gpurun_out/ab_$tag.log" <<'PY'
import json, sys
w, envs, f = sys.argv[1:]
try:
    r = json.loads([l for l in open(f) if l.startswith("{")][-1])
    print(f"{w} [{envs}]: step {r['ms_per_step']:.3f}  search {r['breakdown_ms']['search_topl_softmax']:.3f}  wpsum {r['breakdown_ms']['wpsum']:.3f}  bwd {r['breakdown_ms'].get('backward', 0):.3f}  frac {r['roofline']['frac']:.3f}")
except Exception as e:
    print(w, envs, "FAILED", e); print(open(f).read()[-1500:])
PY
done
