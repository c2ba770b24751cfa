# GPU batch 38: leaner planner head and one-round scans: full suite (incl. whole-config), step overhead, launch list, final lines
O=gpurun_out
timeout 3000 python -m pytest tests -m gpu -x -q > $O/r2_s38_tests.log 2>&1; echo "tests rc=$?" >> $O/r2_s38_tests.log
tail -4 $O/r2_s38_tests.log
python bench.py --steps 20 --warmup 5 > $O/final4_bench_default.json 2> $O/final4_bench_default.err
python bench.py --impl reference --steps 5 --warmup 1 > $O/final4_bench_reference.json 2> $O/final4_bench_reference.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/final4_launches_default.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/final4_launches.log 2>&1
timeout 1500 python tools/shard_sim.py --shards 1,2,4,8 --steps 5 > $O/final4_shard_sim.jsonl 2> $O/final4_shard_sim.err
python - <<'E'
import json,csv
for f in ('default','reference'):
    j=json.loads(open('gpurun_out/final4_bench_%s.json'%f).read().strip().splitlines()[-1])
    print(f, round(j['value'],1), round(j['ms_per_step'],3), j.get('e2e') and round(j['e2e']['value'],1), j.get('roofline') and j['roofline'].get('frac'), j.get('gpu_launches'), j.get('cascade') and j['cascade']['ms_per_call'])
rows=list(csv.reader(open('gpurun_out/final4_launches_default.csv')))
hi=[i for i,r in enumerate(rows) if 'Kernel Name' in r][0]
h=rows[hi]; kn=h.index('Kernel Name'); mv=h.index('Metric Value')
seq=[(r[kn], float(r[mv].replace(',',''))) for r in rows[hi+2:] if len(r)>mv]
big=[i for i,(k,v) in enumerate(seq) if 'tc_search_kernel' in k and v>15e6]
i=big[-1]
for k,v in seq[i-14:i+3]: print(f"{v/1000:10.2f} us  {k[:70]}")
for l in open('gpurun_out/final4_shard_sim.jsonl'):
    if l.startswith('{"shards"'):
        j=json.loads(l); print(j['shards'], j['critical_path_ms'], round(j['speedup_vs_1'],3))
E
