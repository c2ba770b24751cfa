# GPU batch 9: collect + select top-k -- parity, then A/B against the register-list passes
O=gpurun_out
timeout 1500 python -m pytest tests/test_search_gpu.py tests/test_multi_device_gpu.py tests/test_full_size_gpu.py -m gpu -x -q > $O/r2_s09_tests.log 2>&1; echo "rc=$?" >> $O/r2_s09_tests.log
show='import json,sys
for l in sys.stdin:
    l=l.strip()
    if not l.startswith("{"): continue
    j=json.loads(l); r=j["roofline"]
    print(" ms", round(j["ms_per_step"],3), "kernel_sum", round(r["kernel_ms_per_launch"]*r["launches_per_step"],3), "clk", j["clocks"]["sm_mhz"], "e2e", round(j["e2e"]["value"]), j.get("cpu_baseline") and j["cpu_baseline"].get("topk_parity"))'
( for k in 2 5 16 32 64; do for mode in collect lists; do
  echo "k=$k mode=$mode"
  HOMS_B200_TC_TOPK=$mode timeout 600 python bench.py --k $k --steps 5 --warmup 3 2>/dev/null | python -c "$show"
done; done
echo "hek293 k=16 collect"; timeout 900 python bench.py --workload hek293 --k 16 --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "$show"
echo "hek293 k=16 lists"; HOMS_B200_TC_TOPK=lists timeout 900 python bench.py --workload hek293 --k 16 --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "$show"
) > $O/r2_s09_topk_ab.log 2>&1
tail -5 $O/r2_s09_tests.log; cat $O/r2_s09_topk_ab.log
