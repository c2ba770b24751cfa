# GPU batch 34: resident query chunks for CTA pairs (D <= 2048): suite + interleaved A/B
O=gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q --deselect tests/test_whole_config_gpu.py > $O/r2_s34_tests.log 2>&1; echo "rc=$?" >> $O/r2_s34_tests.log
tail -4 $O/r2_s34_tests.log
show='import json,sys
for l in sys.stdin:
    l=l.strip()
    if not l.startswith("{"): continue
    j=json.loads(l); r=j["roofline"]
    print(" ms", round(j["ms_per_step"],4), "kernel", round(r["kernel_ms_per_launch"],4), "clk", j["clocks"]["sm_mhz"], "frac", round(r.get("frac") or 0,4), "e2e", round(j["e2e"]["value"]))'
( for rep in 1 2; do
  echo "D=1024 single+ares rep=$rep"; timeout 600 python bench.py --dim 1024 --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "$show"
  echo "D=1024 pair+ares rep=$rep"; HOMS_B200_TC_PAIR=1 timeout 600 python bench.py --dim 1024 --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "$show"
  echo "D=2048 pair+ares rep=$rep"; timeout 600 python bench.py --dim 2048 --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "$show"
  echo "D=2048 pair streaming rep=$rep"; HOMS_B200_TC_ARES=0 timeout 600 python bench.py --dim 2048 --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "$show"
done
echo "hek293 D=1024 single+ares"; timeout 900 python bench.py --workload hek293 --dim 1024 --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "$show"
echo "hek293 D=1024 pair+ares"; HOMS_B200_TC_PAIR=1 timeout 900 python bench.py --workload hek293 --dim 1024 --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "$show"
echo "hek293 D=2048 pair+ares"; timeout 900 python bench.py --workload hek293 --dim 2048 --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "$show"
echo "hek293 D=2048 pair streaming"; HOMS_B200_TC_ARES=0 timeout 900 python bench.py --workload hek293 --dim 2048 --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "$show"
echo "D=512 single+ares"; timeout 600 python bench.py --dim 512 --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "$show"
echo "D=512 pair+ares"; HOMS_B200_TC_PAIR=1 timeout 600 python bench.py --dim 512 --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "$show"
) > $O/r2_s34_ab_pair_ares.log 2>&1
cat $O/r2_s34_ab_pair_ares.log
