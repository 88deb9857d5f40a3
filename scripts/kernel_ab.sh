#!/bin/bash
# A/B of the search register plans on the GPU box: tests + bench lines per workload.
# usage: scripts/kernel_ab.sh [workloads...]   (writes gpurun_out/ab_*.log)
set -u
mkdir -p gpurun_out
WL=${*:-c4 c2 c5}
for k in stream tiled; do
  for w in $WL; do
    steps=20; [ "$w" = c5 ] && steps=5
    SNLS_SEARCH_KERNEL=$k timeout 300 python bench.py --workload $w --steps $steps --warmup 3 --no-cpu-baseline \
      > gpurun_out/ab_${k}_${w}.log 2>&1
    python - "$k" "$w" <<'PY'
import json, sys
k, w = sys.argv[1:]
try:
    line = [l for l in open(f"gpurun_out/ab_{k}_{w}.log") if l.startswith("{")][-1]
    r = json.loads(line)
    print(f"{k:7s} {w}: step {r['ms_per_step']:.3f} ms  search {r['breakdown_ms']['search_topl_softmax']:.3f}  wpsum {r['breakdown_ms']['wpsum']:.3f}  frac {r['roofline']['frac']:.3f}  e2e {r['e2e']['ms_per_step']:.3f}")
except Exception as e:
    print(k, w, "FAILED", e); print(open(f"gpurun_out/ab_{k}_{w}.log").read()[-1500:])
PY
  done
done
