#!/bin/bash
# usage: scripts/e2e_sweep.sh WORKLOAD CHUNK...  -> device ms, streamed e2e ms, one-clip e2e ms
w=$1; shift
mkdir -p gpurun_out
for c in "$@"; do
  python bench.py --workload $w --steps ${STEPS:-50} --warmup 3 --no-cpu-baseline --pipe-chunk $c > gpurun_out/sweep_${w}_$c.json 2> gpurun_out/sweep_${w}_$c.err
  python - "$w" "$c" <<'PY'
import json, sys
w, c = sys.argv[1:]
r = json.loads([l for l in open(f"gpurun_out/sweep_{w}_{c}.json") if l.startswith("{")][-1])
print(f"{w} chunk {c}: device {r['ms_per_step']:.3f}  e2e streamed {r['e2e']['ms_per_step']:.3f}  one clip {r['e2e']['sync_ms_per_step']:.3f}")
PY
done
