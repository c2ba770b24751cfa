#!/bin/bash
# A/B of encode-kernel builds on the GPU box: HOMS_B200_LIB selects the shared object (development aid)
for lib in "$@"; do
  echo "== $lib"
  HOMS_B200_LIB=$lib python bench.py --workload encode --steps 3 --warmup 3 --no-cpu-baseline --encode-spectra 250000 2>/dev/null | python -c "
import json,sys
j=json.loads(sys.stdin.read()); r=j['roofline']
print('spectra/s %.4g  encode_kernel_ms %.3f  share %.3f  e2e %.4g  clk %s' % (j['value'], r['kernel_ms_per_launch'], r['kernel_share_of_step'], j['e2e']['value'], j['clocks']['sm_mhz']))"
done
