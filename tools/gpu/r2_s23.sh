# GPU batch 23: 64-bit peer FIFO entries, pairs from D = 2048: search suite + sanitizers on the pair form
O=gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q --deselect tests/test_whole_config_gpu.py > $O/r2_s23_tests.log 2>&1; echo "rc=$?" >> $O/r2_s23_tests.log
tail -4 $O/r2_s23_tests.log
timeout 1800 compute-sanitizer --tool memcheck --error-exitcode 9 \
  python -m pytest tests/test_search_gpu.py -m gpu -x -q -k "golden or kernel_forms or index_order or topk_modes" > $O/r2_s23_memcheck.log 2>&1
echo "memcheck rc=$?" >> $O/r2_s23_memcheck.log
timeout 1500 compute-sanitizer --tool racecheck --error-exitcode 9 \
  python -m pytest tests/test_search_gpu.py -m gpu -x -q -k "golden or kernel_forms or index_order" > $O/r2_s23_racecheck.log 2>&1
echo "racecheck rc=$?" >> $O/r2_s23_racecheck.log
tail -3 $O/r2_s23_memcheck.log; grep -c "Race reported" $O/r2_s23_racecheck.log; grep "Race reported\|and " $O/r2_s23_racecheck.log | sed 's/+0x[0-9a-f]*//g' | sort | uniq -c | sort -rn | head -20; tail -3 $O/r2_s23_racecheck.log
show='import json,sys
for l in sys.stdin:
    l=l.strip()
    if not l.startswith("{"): continue
    j=json.loads(l); r=j["roofline"]
    print(" ms", round(j["ms_per_step"],4), "kernel", round(r["kernel_ms_per_launch"],4), "clk", j["clocks"]["sm_mhz"], "frac", round(r.get("frac") or 0,4), "probe", round(r["peak"]), "e2e", round(j["e2e"]["value"]))'
for rep in 1 2; do timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "$show"; done
