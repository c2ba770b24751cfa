#!/bin/bash
# engine crossover for narrow windows: config-2 shape at several tolerances on both engines (development aid)
for tol in ppm:20 ppm:200 da:1 da:5 da:20 da:100; do
  for eng in auto popc; do
    python bench.py --steps 5 --warmup 3 --no-cpu-baseline --tol $tol --engine $eng 2>/dev/null | python -c "
import json,sys
j=json.loads(sys.stdin.read()); r=j['roofline']
print('tol=$tol eng=$eng ms %.3f q/s %.0f kernel_ms %.3f pairs %d' % (j['ms_per_step'], j['value'], r['kernel_ms_per_launch'], j['config']['candidate_pairs_per_step']))"
  done
done
