# GPU batch 31: final suite (incl. whole-config parity) and the default / reference lines of the final build
O=gpurun_out
timeout 3000 python -m pytest tests -m gpu -x -q --durations=6 > $O/r2_s31_tests.log 2>&1; echo "tests rc=$?" >> $O/r2_s31_tests.log
tail -12 $O/r2_s31_tests.log
python bench.py --steps 20 --warmup 5 > $O/final2_bench_default.json 2> $O/final2_bench_default.err
python bench.py --impl reference --steps 5 --warmup 1 > $O/final2_bench_reference.json 2> $O/final2_bench_reference.err
timeout 900 python bench.py --dim 1024 --steps 10 --warmup 3 > $O/final2_bench_dim1024.json 2> $O/final2_bench_dim1024.err
python -c "
import json
for f in ('default','reference','dim1024'):
    j=json.loads(open('gpurun_out/final2_bench_%s.json'%f).read().strip().splitlines()[-1])
    print(f, round(j['value'],1), round(j['ms_per_step'],3), j.get('e2e') and round(j['e2e']['value'],1), j.get('roofline') and j['roofline'].get('frac'), j.get('gpu_launches'))
"
python -c "import __graft_entry__ as g; g.smoke()"
