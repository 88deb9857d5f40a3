#!/bin/bash
# usage: scripts/e2e_ab.sh WORKLOAD CHUNK "ENV=.." ...  -> e2e per env set
w=$1; c=$2; shift 2
mkdir -p gpurun_out
for envs in "$@"; do
  tag=$(echo "$w $c $envs" | tr ' =/' '___')
  env $envs python bench.py --workload $w --steps ${STEPS:-50} --warmup 3 --no-cpu-baseline --pipe-chunk $c > gpurun_out/e2eab_$tag.json 2> gpurun_out/e2eab_$tag.err
  python - "$w" "$c" "$envs" "gpurun_out/e2eab_$tag.json" <<'PY'
import json, sys
w, c, envs, f = sys.argv[1:]
try:
    r = json.loads([l for l in open(f) if l.startswith("{")][-1])
    print(f"{w} chunk {c} [{envs}]: device {r['ms_per_step']:.3f}  e2e streamed {r['e2e']['ms_per_step']:.3f}  one clip {r['e2e']['sync_ms_per_step']:.3f}  launches {r.get('gpu_launches')}")
except Exception as e:
    print(w, c, envs, "FAILED", e); print(open(f.replace('.json', '.err')).read()[-1500:])
PY
done
