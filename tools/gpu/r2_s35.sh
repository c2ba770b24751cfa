# GPU batch 35: config-5 sweep on the final build (resident query chunks at D = 1024)
O=gpurun_out
timeout 3000 python tools/config5_sweep.py > $O/final3_config5_sweep_1gpu.jsonl 2> $O/final3_config5_sweep.err
python - <<'E'
import json
for l in open('gpurun_out/final3_config5_sweep_1gpu.jsonl'):
    l=l.strip()
    if l.startswith('{'):
        j=json.loads(l); print(j['dim'], j['tol'], j['engine'], round(j['ms_per_step'],4), round(j['queries_per_s']), j.get('tensor_tops') and round(j['tensor_tops']), j['parity'])
E
