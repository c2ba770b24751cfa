# development sweep: BASELINE config 5 shapes on one GPU (iprg2012-sized library)
for cfg in "1024 da:500" "2048 da:500" "4096 da:500" "8192 da:500" "16384 da:500" "1024 ppm:20" "2048 ppm:20" "4096 ppm:20" "8192 ppm:20" "16384 ppm:20"; do set -- $cfg
 for eng in auto; do
  python bench.py --dim $1 --tol $2 --engine $eng --no-cpu-baseline --steps 5 2>/dev/null | python -c "import json,sys; j=json.loads(sys.stdin.read()); r=j['roofline']; print('D=$1 tol=$2 eng=$eng', 'ms', round(j['ms_per_step'],3), 'q/s', round(j['value']), 'kernel_ms', round(r['kernel_ms_per_launch'],3), 'share', round(r['kernel_share_of_step'],3), 'frac', round(r['frac'],3), 'clk', j['clocks']['sm_mhz'])"
 done
done
