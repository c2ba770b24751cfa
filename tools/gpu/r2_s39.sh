# GPU batch 39: default / reference lines and launch list of the final build
O=gpurun_out
python bench.py --steps 20 --warmup 5 > $O/final5_bench_default.json 2> $O/final5_bench_default.err
python bench.py --impl reference --steps 5 --warmup 1 > $O/final5_bench_reference.json 2> $O/final5_bench_reference.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/final5_launches_default.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/final5_launches.log 2>&1
timeout 600 python -m pytest tests/test_search_gpu.py tests/test_mgf_gpu.py -m gpu -x -q > $O/r2_s39_tests.log 2>&1; tail -2 $O/r2_s39_tests.log
python - <<'E'
import json
for f in ('default','reference'):
    j=json.loads(open('gpurun_out/final5_bench_%s.json'%f).read().strip().splitlines()[-1])
    print(f, round(j['value'],1), round(j['ms_per_step'],3), j.get('e2e') and round(j['e2e']['value'],1), j.get('roofline') and j['roofline'].get('frac'), j.get('gpu_launches'), j.get('cascade') and j['cascade']['ms_per_call'])
E
python -c "import __graft_entry__ as g; g.smoke()"
