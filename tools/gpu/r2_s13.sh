# GPU batch 13: CTA-pair kernel with relaxed remote arrives: parity subset, interleaved A/B; collect buffer statistics;
# bulk-copy staged gather microbenchmark
O=gpurun_out
HOMS_B200_TC_PAIR=1 timeout 1500 python -m pytest tests/test_search_gpu.py -m gpu -x -q -k "tensor or auto or topk or planning or tight" > $O/r2_s13_tests_pair.log 2>&1; echo "rc=$?" >> $O/r2_s13_tests_pair.log
tail -5 $O/r2_s13_tests_pair.log
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
) > $O/r2_s13_pair_ab.log 2>&1
cat $O/r2_s13_pair_ab.log
( for k in 5 9 16; do echo "collect k=$k"; HOMS_B200_TC_DEBUG=1 HOMS_B200_TC_TOPK=collect timeout 600 python bench.py --k $k --steps 1 --warmup 1 --no-cpu-baseline 2>&1 | grep "tc collect" | tail -2; done ) > $O/r2_s13_collect_stats.log 2>&1
cat $O/r2_s13_collect_stats.log
timeout 600 tools/l2_gather_bench > $O/r2_s13_l2_gather.txt 2>&1; grep "TMA\|BEST\|status" $O/r2_s13_l2_gather.txt
