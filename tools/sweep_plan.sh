# development sweep: work-item length under the dynamic work queue (items per SM -> strip length)
for cfg in "400 8" "100 32" "200 32" "300 32" "600 32" "800 32" "1600 32" "400 8"; do set -- $cfg
  for w in "" "--workload hek293"; do
    HOMS_B200_TC_ITEMS_PER_SM=$1 HOMS_B200_TC_MAX_STRIP=$2 python bench.py --no-cpu-baseline --steps 3 $w 2>/dev/null | python -c "import json,sys; j=json.loads(sys.stdin.read()); print('IPS=$1 maxstrip=$2 $w ms', round(j['ms_per_step'],2), 'kernel', round(j['roofline']['kernel_ms_per_launch'],2), 'clk', j['clocks']['sm_mhz'])"
  done
done
