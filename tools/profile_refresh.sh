#!/bin/bash
# profile refresh after the device planner / top-k (development aid)
O=gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/refresh_launches_tensor_fp4.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline > $O/refresh_launches.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:tc_search_kernel -c 1 -f -o $O/refresh_search_full \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $O/refresh_ncu_search.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:tc_search_kernel -c 1 -f -o $O/refresh_search_k5_full \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline --k 5 > $O/refresh_ncu_search_k5.log 2>&1
python bench.py --steps 5 --warmup 3 > $O/refresh_bench_default.json 2> $O/refresh_bench_default.err
python bench.py --steps 5 --warmup 3 --k 5 --no-cpu-baseline > $O/refresh_bench_k5.json 2> $O/refresh_bench_k5.err
python bench.py --steps 5 --warmup 3 --k 16 --no-cpu-baseline > $O/refresh_bench_k16.json 2> $O/refresh_bench_k16.err
python bench.py --impl reference --steps 2 --warmup 1 > $O/refresh_bench_reference.json 2> $O/refresh_bench_reference.err
