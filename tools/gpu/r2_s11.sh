# GPU batch 11: CTA-pair probe (cta_group::2 semantics + issue rate under the power cap), own radix sort in
# the search step and build_index (parity suite), top-k policy (lists <= 8 < collect)
O=gpurun_out
timeout 300 tools/tc_pair_probe 0.5 > $O/r2_s11_pair_probe.txt 2>&1; echo "rc=$?" >> $O/r2_s11_pair_probe.txt
timeout 2400 python -m pytest tests -m gpu -x -q --deselect tests/test_whole_config_gpu.py > $O/r2_s11_tests.log 2>&1; echo "rc=$?" >> $O/r2_s11_tests.log
timeout 600 python bench.py --steps 10 --warmup 3 > $O/r2_s11_bench_default.json 2> $O/r2_s11_bench_default.err
show='import json,sys
for l in sys.stdin:
    l=l.strip()
    if not l.startswith("{"): continue
    j=json.loads(l); r=j["roofline"]
    print(" ms", round(j["ms_per_step"],3), "kernel_sum", round(r["kernel_ms_per_launch"]*r["launches_per_step"],3), "clk", j["clocks"]["sm_mhz"], "e2e", round(j["e2e"]["value"]), j.get("cpu_baseline") and j["cpu_baseline"].get("topk_parity"))'
( for k in 8 9; do echo "k=$k"; timeout 600 python bench.py --k $k --steps 5 --warmup 3 2>/dev/null | python -c "$show"; done
  echo "20 ppm"; timeout 600 python bench.py --tol ppm:20 --steps 20 --warmup 3 2>/dev/null | python -c "$show"
) > $O/r2_s11_misc.log 2>&1
cat $O/r2_s11_pair_probe.txt; tail -5 $O/r2_s11_tests.log; cat $O/r2_s11_misc.log; python - <<'E'
import json
j=json.loads(open("gpurun_out/r2_s11_bench_default.json").read().strip().splitlines()[-1])
print(j["ms_per_step"], j["value"], j["e2e"]["value"], j["roofline"]["frac"], j["gpu_launches"], j["cascade"]["ms_per_call"])
E
