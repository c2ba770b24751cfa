# GPU batch 44: final build with the eviction hints off: search suite, ncu full capture, default / reference lines, launch list
O=gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q --deselect tests/test_whole_config_gpu.py > $O/r2_s44_tests.log 2>&1; echo "rc=$?" >> $O/r2_s44_tests.log
tail -3 $O/r2_s44_tests.log
ncu --set full --clock-control none --import-source on -k regex:tc_search_kernel -s 3 -c 1 -f -o $O/final6_search_top1 \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $O/final6_ncu_top1.log 2>&1
ncu -i $O/final6_search_top1.ncu-rep --page raw --csv > $O/final6_search_top1_raw.csv 2>/dev/null
python tools/ncu_summary.py $O/final6_search_top1_raw.csv > $O/final6_search_top1_ncu.csv
head -22 $O/final6_search_top1_ncu.csv
python bench.py --steps 20 --warmup 5 > $O/final6_bench_default.json 2> $O/final6_bench_default.err
python bench.py --impl reference --steps 5 --warmup 1 > $O/final6_bench_reference.json 2> $O/final6_bench_reference.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/final6_launches_default.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/final6_launches.log 2>&1
python - <<'E'
import json
for f in ('default','reference'):
    j=json.loads(open('gpurun_out/final6_bench_%s.json'%f).read().strip().splitlines()[-1])
    print(f, round(j['value'],1), round(j['ms_per_step'],3), j.get('e2e') and round(j['e2e']['value'],1), j.get('roofline') and (j['roofline'].get('frac'), j['roofline'].get('traffic_over_compulsory')), j.get('gpu_launches'))
E
