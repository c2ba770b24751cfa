# development check: group size on the config-3 prefix (4.3 M rows) and config 2
run() { python bench.py --no-cpu-baseline --steps 3 "$@" 2>/dev/null | python -c "import json,sys; j=json.loads(sys.stdin.read()); print(' ms', round(j['ms_per_step'],2), 'kernel', round(j['roofline']['kernel_ms_per_launch'],2), 'clk', j['clocks']['sm_mhz'])"; }
for g in 24 32 48 64 80; do
  echo "G=$g hek293"; HOMS_B200_TC_GROUP=$g run --workload hek293
  echo "G=$g iprg2012"; HOMS_B200_TC_GROUP=$g run
done
