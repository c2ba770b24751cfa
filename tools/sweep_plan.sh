# development sweep: planner knobs (group of query tiles, max strip length) under the dynamic work queue
for cfg in "12 8" "24 8" "32 8" "48 8" "64 8" "125 8" "32 4" "32 16" "12 8"; do set -- $cfg
  for k in 1 5; do
    HOMS_B200_TC_GROUP=$1 HOMS_B200_TC_MAX_STRIP=$2 python bench.py --no-cpu-baseline --steps 5 --k $k 2>/dev/null | python -c "import json,sys; j=json.loads(sys.stdin.read()); print('G=$1 strip=$2 k=$k ms', round(j['ms_per_step'],2), 'kernel', round(j['roofline']['kernel_ms_per_launch'],2), 'clk', j['clocks']['sm_mhz'])"
  done
done
