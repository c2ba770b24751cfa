# GPU batch 16: direct engine with several short rows side by side in the warp (D <= 2048): full suite, 20 ppm timings
O=gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q --deselect tests/test_whole_config_gpu.py > $O/r2_s16_tests.log 2>&1; echo "rc=$?" >> $O/r2_s16_tests.log
tail -4 $O/r2_s16_tests.log
show='import json,sys
for l in sys.stdin:
    l=l.strip()
    if not l.startswith("{"): continue
    j=json.loads(l); r=j["roofline"]
    print(" ms", round(j["ms_per_step"],4), "kernel", round(r["kernel_ms_per_launch"],4), "x", r["launches_per_step"], "clk", j["clocks"]["sm_mhz"], "e2e", round(j["e2e"]["value"]), j["config"]["workload"][:60])'
( for d in 1024 2048 4096; do echo "hek293 D=$d 20 ppm"; timeout 900 python bench.py --workload hek293 --dim $d --tol ppm:20 --steps 20 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "$show"; done
  for d in 1024 2048; do echo "iprg D=$d 20 ppm k=5"; timeout 900 python bench.py --dim $d --tol ppm:20 --k 5 --steps 20 --warmup 3 2>/dev/null | python -c "$show"; done
) > $O/r2_s16_direct_small.log 2>&1
cat $O/r2_s16_direct_small.log
