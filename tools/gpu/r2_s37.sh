# GPU batch 37: warp-parallel plan_items: suite, step overhead
O=gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q --deselect tests/test_whole_config_gpu.py > $O/r2_s37_tests.log 2>&1; echo "rc=$?" >> $O/r2_s37_tests.log
tail -4 $O/r2_s37_tests.log
show='import json,sys
for l in sys.stdin:
    l=l.strip()
    if not l.startswith("{"): continue
    j=json.loads(l); r=j["roofline"]
    print(" ms", round(j["ms_per_step"],4), "kernel", round(r["kernel_ms_per_launch"],4), "overhead", round(j["ms_per_step"]-r["kernel_ms_per_launch"]*r["launches_per_step"],4), "clk", j["clocks"]["sm_mhz"])'
for rep in 1 2; do timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "$show"; done
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/r2_s37_launches_default.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/r2_s37_launches.log 2>&1
grep "tc_plan_items" $O/r2_s37_launches_default.csv | tail -2 | awk -F'","' '{print $5, $NF}' | cut -c 1-60,100-
