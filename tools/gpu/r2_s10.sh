# GPU batch 10 (re-entry): full gpu suite, default bench, collect vs lists top-k A/B
O=gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q > $O/r2_s10_tests.log 2>&1; echo "rc=$?" >> $O/r2_s10_tests.log
timeout 600 python bench.py > $O/r2_s10_bench_default.json 2> $O/r2_s10_bench_default.err
show='import json,sys
for l in sys.stdin:
    l=l.strip()
    if not l.startswith("{"): continue
    j=json.loads(l); r=j["roofline"]
    print(" ms", round(j["ms_per_step"],3), "kernel_sum", round(r["kernel_ms_per_launch"]*r["launches_per_step"],3), "clk", j["clocks"]["sm_mhz"], "e2e", round(j["e2e"]["value"]), j.get("cpu_baseline") and j["cpu_baseline"].get("topk_parity"))'
( for k in 2 5 16 32 64; do for mode in collect lists; do
  echo "k=$k mode=$mode"
  HOMS_B200_TC_TOPK=$mode timeout 600 python bench.py --k $k --steps 5 --warmup 3 2>/dev/null | python -c "$show"
done; done ) > $O/r2_s10_topk_ab.log 2>&1
tail -5 $O/r2_s10_tests.log; cat $O/r2_s10_bench_default.json; cat $O/r2_s10_topk_ab.log
