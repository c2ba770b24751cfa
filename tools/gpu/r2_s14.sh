# GPU batch 14: own scan in the MGF parser + per-chunk floor refresh (full suite), pair kernel with the fence-free FIFO
O=gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q --deselect tests/test_whole_config_gpu.py > $O/r2_s14_tests.log 2>&1; echo "rc=$?" >> $O/r2_s14_tests.log
tail -4 $O/r2_s14_tests.log
HOMS_B200_TC_PAIR=1 timeout 1500 python -m pytest tests/test_search_gpu.py tests/test_multi_device_gpu.py -m gpu -x -q > $O/r2_s14_tests_pair.log 2>&1; echo "rc=$?" >> $O/r2_s14_tests_pair.log
tail -4 $O/r2_s14_tests_pair.log
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
for pair in 0 1; do echo "D=1024 pair=$pair"; HOMS_B200_TC_PAIR=$pair timeout 900 python bench.py --dim 1024 --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "$show"; done
for pair in 0 1; do echo "D=16384 pair=$pair"; HOMS_B200_TC_PAIR=$pair timeout 900 python bench.py --dim 16384 --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "$show"; done
) > $O/r2_s14_pair_ab.log 2>&1
cat $O/r2_s14_pair_ab.log
( for k in 2 5 8 16 64; do for mode in collect lists; do echo "k=$k mode=$mode"; HOMS_B200_TC_DEBUG=1 HOMS_B200_TC_TOPK=$mode timeout 600 python bench.py --k $k --steps 5 --warmup 3 --no-cpu-baseline 2> $O/err.txt | python -c "$show"; grep "tc collect" $O/err.txt | tail -1; done; done ) > $O/r2_s14_topk_ab.log 2>&1
cat $O/r2_s14_topk_ab.log
