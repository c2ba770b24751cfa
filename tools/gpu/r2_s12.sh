# GPU batch 12: CTA-pair search kernel (HOMS_B200_TC_PAIR=1): parity, then interleaved A/B; collect-mode buffer size at small k
O=gpurun_out
HOMS_B200_TC_PAIR=1 timeout 1500 python -m pytest tests/test_search_gpu.py tests/test_multi_device_gpu.py -m gpu -x -q > $O/r2_s12_tests_pair.log 2>&1; echo "rc=$?" >> $O/r2_s12_tests_pair.log
tail -5 $O/r2_s12_tests_pair.log
show='import json,sys
for l in sys.stdin:
    l=l.strip()
    if not l.startswith("{"): continue
    j=json.loads(l); r=j["roofline"]
    print(" ms", round(j["ms_per_step"],3), "kernel", round(r["kernel_ms_per_launch"],3), "x", r["launches_per_step"], "clk", j["clocks"]["sm_mhz"], "frac", round(r["frac"],4), "e2e", round(j["e2e"]["value"]), j.get("cpu_baseline") and j["cpu_baseline"].get("topk_parity"))'
( for rep in 1 2; do for pair in 0 1; do
  echo "pair=$pair rep=$rep"
  HOMS_B200_TC_PAIR=$pair timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "$show"
done; done
for pair in 0 1; do echo "hek293 pair=$pair"; HOMS_B200_TC_PAIR=$pair timeout 900 python bench.py --workload hek293 --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "$show"; done
for pair in 0 1; do echo "D=1024 pair=$pair"; HOMS_B200_TC_PAIR=$pair timeout 900 python bench.py --dim 1024 --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "$show"; done
) > $O/r2_s12_pair_ab.log 2>&1
cat $O/r2_s12_pair_ab.log
( for ccap in 1024 4096; do for k in 5 9; do echo "collect k=$k ccap=$ccap"; HOMS_B200_TC_TOPK=collect HOMS_B200_TC_CCAP=$ccap timeout 600 python bench.py --k $k --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "$show"; done; done ) > $O/r2_s12_ccap.log 2>&1
cat $O/r2_s12_ccap.log
