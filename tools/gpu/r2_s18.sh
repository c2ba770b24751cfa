# GPU batch 18: single-thread roles entered through elect.sync (no per-instruction waterfall loops around UBLKCP /
# UTCOMMA / UTCBAR); radix selection of the top max_peaks in the preprocess kernel
O=gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q --deselect tests/test_whole_config_gpu.py > $O/r2_s18_tests.log 2>&1; echo "rc=$?" >> $O/r2_s18_tests.log
tail -4 $O/r2_s18_tests.log
show='import json,sys
for l in sys.stdin:
    l=l.strip()
    if not l.startswith("{"): continue
    j=json.loads(l); r=j["roofline"]
    print(" ms", round(j["ms_per_step"],4), "kernel", round(r["kernel_ms_per_launch"],4), "x", r["launches_per_step"], "clk", j["clocks"]["sm_mhz"], "frac", round(r.get("frac") or 0,4), "e2e", round(j["e2e"]["value"]), j["config"]["workload"][:50])'
( for rep in 1 2; do echo "default rep=$rep"; timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "$show"; done
  echo "k=16"; timeout 600 python bench.py --k 16 --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "$show"
  for d in 1024 2048 4096 16384; do echo "D=$d"; timeout 900 python bench.py --dim $d --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "$show"; done
  echo "hek293"; timeout 900 python bench.py --workload hek293 --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "$show"
  echo "encode max_peaks=50"; timeout 900 python bench.py --workload encode --encode-spectra 2000000 --encode-max-peaks 50 --steps 3 --warmup 3 2>/dev/null | python -c "$show"
  echo "encode max_peaks=150"; timeout 900 python bench.py --workload encode --encode-spectra 2000000 --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "$show"
) > $O/r2_s18_elect.log 2>&1
cat $O/r2_s18_elect.log
