#!/bin/bash
# Re-measure everything profiles/ holds, on the GPU box:
#   gpurun -- scripts/refresh_profiles.sh TAG
# bench lines (c4 default + c2/c3/c5 + c4 with 8 videos per GPU + the reference arm), the c4
# launch list, one ncu --set full capture of the c4 search and wpsum kernels (summarised
# here), the c5 search DRAM traffic, compute-sanitizer over the parity tests.
tag=${1:-r02}
o=gpurun_out
mkdir -p $o
python bench.py > $o/${tag}_bench_c4.json 2> $o/${tag}_bench_c4.err
for w in c2 c3 c5; do
  python bench.py --workload $w > $o/${tag}_bench_$w.json 2> $o/${tag}_bench_$w.err
done
python bench.py --workload c3 --deterministic --no-cpu-baseline > $o/${tag}_bench_c3_deterministic.json 2>/dev/null
python bench.py --videos-per-gpu 8 --steps 10 --no-cpu-baseline > $o/${tag}_bench_c4_8videos.json 2> /dev/null
python bench.py --impl reference > $o/${tag}_bench_reference_c4.json 2> $o/${tag}_bench_reference_c4.err
ncu --metrics gpu__time_duration.sum --clock-control none -s 18 -c 30 --csv --log-file $o/${tag}_launches_c4.csv \
  python bench.py --steps 10 --warmup 5 --no-cpu-baseline > /dev/null 2>&1
python scripts/launch_shares.py $o/${tag}_launches_c4.csv > $o/${tag}_launches_c4.txt
scripts/ncu_capture.sh $tag c4 'regex:search_tiled_kernel|wpsum_query_kernel' 2
scripts/ncu_capture.sh $tag c3 'regex:search_tiled_kernel|wpsum_patch|wpsum_combine|search_bwd_rows|wpsum_bwd' 5
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
  -k regex:search_tiled -s 1 -c 1 python bench.py --workload c5 --steps 1 --warmup 3 --no-cpu-baseline 2>/dev/null \
  | grep -E "dram__|gpu__time" > $o/${tag}_c5_search_dram.txt
{
  echo "# compute-sanitizer over the GPU parity tests on B200 ($tag)"
  for t in memcheck racecheck synccheck; do
    tests="tests/test_gpu_kernels.py tests/test_gpu_search.py tests/test_gpu_backward.py tests/test_gpu_c3.py tests/test_gpu_wpsum_patch.py"
    [ $t = memcheck ] && tests="$tests tests/test_gpu_aggregate.py tests/test_gpu_pipeline.py tests/test_gpu_shard.py tests/test_gpu_align.py tests/test_gpu_robustness.py"
    compute-sanitizer --tool $t --error-exitcode 9 python -m pytest -q -x $tests > $o/san_$t.log 2>&1
    echo "$t rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|passed|failed' $o/san_$t.log | tail -2 | tr '\n' ' ')"
  done
} > $o/${tag}_sanitizer.txt
