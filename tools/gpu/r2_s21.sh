# GPU batch 21: CTA pairs by default for D >= 8192 + lean producer loop: full suite incl. whole-config parity, pair threshold
O=gpurun_out
timeout 3000 python -m pytest tests -m gpu -x -q > $O/r2_s21_tests.log 2>&1; echo "rc=$?" >> $O/r2_s21_tests.log
tail -4 $O/r2_s21_tests.log
show='import json,sys
for l in sys.stdin:
    l=l.strip()
    if not l.startswith("{"): continue
    j=json.loads(l); r=j["roofline"]
    print(" ms", round(j["ms_per_step"],4), "kernel", round(r["kernel_ms_per_launch"],4), "clk", j["clocks"]["sm_mhz"], "frac", round(r.get("frac") or 0,4), "probe", round(r["peak"]), "e2e", round(j["e2e"]["value"]))'
( for rep in 1 2; do for pair in 0 1; do
  echo "pair=$pair rep=$rep"
  HOMS_B200_TC_PAIR=$pair timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "$show"
done; done
for args in "--dim 2048" "--dim 4096" "--k 16" "--workload hek293 --dim 4096"; do for pair in 0 1; do
  echo "pair=$pair $args"
  HOMS_B200_TC_PAIR=$pair timeout 900 python bench.py $args --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "$show"
done; done ) > $O/r2_s21_ab_pair.log 2>&1
cat $O/r2_s21_ab_pair.log
