# GPU batch 6: new planner defaults (B evict_first, single group when it fits, byte-sized items): tests + dims
O=gpurun_out
timeout 1200 python -m pytest tests/test_search_gpu.py tests/test_multi_device_gpu.py tests/test_full_size_gpu.py -m gpu -x -q > $O/r2_s06_tests.log 2>&1; echo "rc=$?" >> $O/r2_s06_tests.log
show='import json,sys
for l in sys.stdin:
    l=l.strip()
    if not l.startswith("{"): continue
    j=json.loads(l); r=j["roofline"]
    print(" ms", round(j["ms_per_step"],3), "kernel", round(r["kernel_ms_per_launch"],3), "frac", round(r["frac"],3), "clk", j["clocks"]["sm_mhz"], j["clocks"]["reasons"], "e2e", round(j["e2e"]["value"]))'
( for D in 1024 2048 4096 8192 16384; do
  echo "dim=$D"
  timeout 600 python bench.py --dim $D --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "$show"
done
echo "hek293"; timeout 900 python bench.py --workload hek293 --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "$show"
for k in 5 16; do echo "k=$k"; timeout 600 python bench.py --k $k --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "$show"; done
) > $O/r2_s06_dims.log 2>&1
tail -3 $O/r2_s06_tests.log; cat $O/r2_s06_dims.log
