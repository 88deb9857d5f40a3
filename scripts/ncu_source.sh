#!/bin/bash
# Per-source-line instruction counts and stall samples of one kernel (GPU box):
#   scripts/ncu_source.sh TAG WORKLOAD 'regex:kernel'  -> gpurun_out/TAG_src.csv (+ _sass.csv)
tag=$1; w=$2; k=$3; shift 3
o=gpurun_out; mkdir -p $o
ncu --set full --clock-control none --import-source on -k "$k" -s 2 -c 1 -o $o/${tag}_src -f \
  python bench.py --workload $w --steps 2 --warmup 3 --no-cpu-baseline "$@" > /dev/null 2>&1
ncu -i $o/${tag}_src.ncu-rep --page source --csv --print-source cuda > $o/${tag}_src.csv 2>/dev/null
ncu -i $o/${tag}_src.ncu-rep --page source --csv --print-source sass > $o/${tag}_sass.csv 2>/dev/null
rm -f $o/${tag}_src.ncu-rep
