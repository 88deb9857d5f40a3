#!/bin/bash
# One ncu --set full capture of the named kernels of a bench workload, summarised (on the GPU
# box):  scripts/ncu_capture.sh TAG WORKLOAD 'regex:kernelA|kernelB' [COUNT] [extra bench args]
tag=$1; w=$2; k=$3; n=${4:-4}; shift 4
o=gpurun_out
mkdir -p $o
ncu --set full --clock-control none --import-source on -k "$k" -s 2 -c $n -o $o/${tag}_ncu_$w -f \
  python bench.py --workload $w --steps 2 --warmup 3 --no-cpu-baseline "$@" > /dev/null 2>&1
python scripts/ncu_summary.py $o/${tag}_ncu_$w.ncu-rep > $o/${tag}_ncu_$w.txt
ncu -i $o/${tag}_ncu_$w.ncu-rep --page raw --csv > $o/${tag}_ncu_${w}_raw.csv 2>/dev/null
rm -f $o/${tag}_ncu_$w.ncu-rep
