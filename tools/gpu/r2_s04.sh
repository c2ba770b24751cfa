# GPU batch 4: more planner/hint variants, config 5 sweep on the 4.3 M-row library, config 3 full with the CPU baseline
O=gpurun_out
show='import json,sys
for l in sys.stdin:
    l=l.strip()
    if not l.startswith("{"): continue
    j=json.loads(l); r=j["roofline"]
    print(" ms", round(j["ms_per_step"],3), "kernel", round(r["kernel_ms_per_launch"],3), "frac", round(r["frac"],3), "clk", j["clocks"]["sm_mhz"], j["clocks"]["reasons"], "e2e", round(j["e2e"]["value"]))'
( for H in 0 2; do for GMB in 64 128; do for STRIP in 8 16; do
  echo "hints=$H group_mb=$GMB max_strip=$STRIP"
  HOMS_B200_TC_L2_HINTS=$H HOMS_B200_TC_GROUP_MB=$GMB HOMS_B200_TC_MAX_STRIP=$STRIP timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "$show"
done; done; done
for H in 0 2; do for GMB in 32 64; do
  echo "hek293 hints=$H group_mb=$GMB"
  HOMS_B200_TC_L2_HINTS=$H HOMS_B200_TC_GROUP_MB=$GMB timeout 900 python bench.py --workload hek293 --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "$show"
done; done
for H in 0 2; do for GMB in 32 64; do for D in 1024 16384; do
  echo "dim=$D hints=$H group_mb=$GMB"
  HOMS_B200_TC_L2_HINTS=$H HOMS_B200_TC_GROUP_MB=$GMB timeout 600 python bench.py --dim $D --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "$show"
done; done; done ) > $O/r2_s04_hints_sweep2.log 2>&1
timeout 2400 python tools/config5_sweep.py > $O/r2_s04_config5_sweep.jsonl 2> $O/r2_s04_config5_sweep.err
timeout 1800 python bench.py --workload hek293_full --steps 2 --warmup 3 > $O/r2_s04_bench_hek293_full.json 2> $O/r2_s04_bench_hek293_full.err
tail -30 $O/r2_s04_hints_sweep2.log
