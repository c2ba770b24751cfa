# GPU batch 32: warp-cooperative window bounds (32 probes per round): suite + narrow-window timings
O=gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q --deselect tests/test_whole_config_gpu.py > $O/r2_s32_tests.log 2>&1; echo "rc=$?" >> $O/r2_s32_tests.log
tail -4 $O/r2_s32_tests.log
show='import json,sys
for l in sys.stdin:
    l=l.strip()
    if not l.startswith("{"): continue
    j=json.loads(l); r=j["roofline"]
    print(" ms", round(j["ms_per_step"],4), "kernel", round(r["kernel_ms_per_launch"],4), "clk", j["clocks"]["sm_mhz"], "e2e", round(j["e2e"]["value"]), "cascade", j.get("cascade") and round(j["cascade"]["ms_per_call"],3))'
for args in "--tol ppm:20" "--workload hek293 --tol ppm:20 --dim 1024" "--workload hek293 --tol ppm:20" ""; do echo "bench $args"; timeout 900 python bench.py $args --steps 20 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "$show"; done
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $O/r2_s32_launches_ppm20.csv \
  python bench.py --tol ppm:20 --steps 2 --warmup 1 --no-cpu-baseline > $O/r2_s32_launches.log 2>&1
grep -c "bounds_kernel" $O/r2_s32_launches_ppm20.csv; grep "bounds_kernel" $O/r2_s32_launches_ppm20.csv | tail -2 | cut -c 1-60,200-
