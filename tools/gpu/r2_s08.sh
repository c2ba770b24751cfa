# GPU batch 8: final evidence of round 2 -- suite, default / reference bench lines, launch list, ncu --set full, sanitizer
O=gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q --durations=8 > $O/r2_s08_tests.log 2>&1; echo "tests rc=$?" >> $O/r2_s08_tests.log
python bench.py --steps 20 --warmup 5 > $O/r2_s08_bench_default.json 2> $O/r2_s08_bench_default.err
python bench.py --impl reference --steps 5 --warmup 1 > $O/r2_s08_bench_reference.json 2> $O/r2_s08_bench_reference.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/r2_s08_launches_default.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/r2_s08_launches.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:tc_search_kernel -s 3 -c 1 -f -o $O/r2_s08_search_full \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $O/r2_s08_ncu_search.log 2>&1
ncu -i $O/r2_s08_search_full.ncu-rep --page raw --csv > $O/r2_s08_search_full_raw.csv 2>/dev/null
ncu --set full --clock-control none --import-source on -k regex:tc_search_kernel -s 3 -c 1 -f -o $O/r2_s08_search_k32_full \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline --k 32 > $O/r2_s08_ncu_search_k32.log 2>&1
ncu -i $O/r2_s08_search_k32_full.ncu-rep --page raw --csv > $O/r2_s08_search_k32_full_raw.csv 2>/dev/null
timeout 1500 compute-sanitizer --tool memcheck --error-exitcode 9 \
  python -m pytest tests/test_search_gpu.py tests/test_multi_device_gpu.py tests/test_pipeline_gpu.py -m gpu -x -q \
  -k "golden or known_answers or topk or group_search or group_raw or query_file or engine_selection" > $O/r2_s08_memcheck.log 2>&1
echo "memcheck rc=$?" >> $O/r2_s08_memcheck.log
timeout 1500 compute-sanitizer --tool racecheck --error-exitcode 9 \
  python -m pytest tests/test_search_gpu.py -m gpu -x -q -k "golden or topk_many" > $O/r2_s08_racecheck.log 2>&1
echo "racecheck rc=$?" >> $O/r2_s08_racecheck.log
tail -4 $O/r2_s08_tests.log; tail -2 $O/r2_s08_memcheck.log; tail -2 $O/r2_s08_racecheck.log
