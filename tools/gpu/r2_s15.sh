# GPU batch 15: pair kernel with the fence-free, self-validating FIFO (parity + A/B); L2 prefetch of the next row tile (A/B)
O=gpurun_out
HOMS_B200_TC_PAIR=1 timeout 1500 python -m pytest tests/test_search_gpu.py tests/test_multi_device_gpu.py -m gpu -x -q > $O/r2_s15_tests_pair.log 2>&1; echo "rc=$?" >> $O/r2_s15_tests_pair.log
tail -4 $O/r2_s15_tests_pair.log
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
) > $O/r2_s15_pair_ab.log 2>&1
cat $O/r2_s15_pair_ab.log
( for rep in 1 2; do for pf in 0 1 8; do
  echo "prefetch=$pf rep=$rep"
  if [ $pf = 0 ]; then timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "$show"; else
  HOMS_B200_TC_PREFETCH=$pf timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "$show"; fi
done; done
for pf in 0 8; do echo "hek293 prefetch=$pf"; if [ $pf = 0 ]; then timeout 900 python bench.py --workload hek293 --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "$show"; else HOMS_B200_TC_PREFETCH=$pf timeout 900 python bench.py --workload hek293 --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "$show"; fi; done
) > $O/r2_s15_prefetch_ab.log 2>&1
cat $O/r2_s15_prefetch_ab.log
