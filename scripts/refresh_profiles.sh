#!/bin/bash
# Re-measure everything profiles/ holds, on the GPU box:
#   gpurun -- scripts/refresh_profiles.sh TAG
# bench lines (c4 default + c2/c3/c5 + the reference arm), the c4 launch list, one
# ncu --set full capture of the c4 search and wpsum kernels (summarised here), sanitizers.
tag=${1:-r01}
o=gpurun_out
mkdir -p $o
python bench.py > $o/${tag}_bench_c4.json 2> $o/${tag}_bench_c4.err
for w in c2 c3 c5; do
  python bench.py --workload $w > $o/${tag}_bench_$w.json 2> $o/${tag}_bench_$w.err
done
python bench.py --impl reference > $o/${tag}_bench_reference_c4.json 2> $o/${tag}_bench_reference_c4.err
ncu --metrics gpu__time_duration.sum --clock-control none -s 18 -c 30 --csv --log-file $o/${tag}_launches_c4.csv \
  python bench.py --steps 10 --warmup 5 --no-cpu-baseline > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:'search_tiled_kernel|wpsum_query_kernel' -s 4 -c 2 \
  -o $o/${tag}_ncu_c4 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
python scripts/ncu_summary.py $o/${tag}_ncu_c4.ncu-rep > $o/${tag}_ncu_c4.txt
rm -f $o/${tag}_ncu_c4.ncu-rep
{
  echo "# compute-sanitizer over the GPU parity tests on B200 ($tag)"
  for t in memcheck racecheck synccheck; do
    tests="tests/test_gpu_kernels.py tests/test_gpu_search.py tests/test_gpu_backward.py"
    [ $t = memcheck ] && tests="$tests tests/test_gpu_aggregate.py tests/test_gpu_pipeline.py tests/test_gpu_shard.py tests/test_gpu_align.py"
    compute-sanitizer --tool $t --error-exitcode 9 python -m pytest -q -x $tests > $o/san_$t.log 2>&1
    echo "$t rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|passed|failed' $o/san_$t.log | tail -2 | tr '\n' ' ')"
  done
} > $o/${tag}_sanitizer.txt
python scripts/launch_shares.py $o/${tag}_launches_c4.csv > $o/${tag}_launches_c4.txt
