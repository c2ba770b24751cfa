# GPU batch 24: queries ordered by window start + end (tight union windows): suite, interleaved A/B against start order
O=gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q --deselect tests/test_whole_config_gpu.py > $O/r2_s24_tests.log 2>&1; echo "rc=$?" >> $O/r2_s24_tests.log
tail -4 $O/r2_s24_tests.log
show='import json,sys
for l in sys.stdin:
    l=l.strip()
    if not l.startswith("{"): continue
    j=json.loads(l); r=j["roofline"]
    print(" ms", round(j["ms_per_step"],4), "kernel", round(r["kernel_ms_per_launch"],4), "clk", j["clocks"]["sm_mhz"], "frac", round(r.get("frac") or 0,4), "e2e", round(j["e2e"]["value"]), "cascade", j.get("cascade") and round(j["cascade"]["ms_per_call"],3))'
( for rep in 1 2 3; do for lib in build_ab/libstartsort.so ""; do
  echo "lib=${lib:-sum-order} rep=$rep"
  HOMS_B200_LIB=${lib:+$PWD/$lib} timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "$show"
done; done
for args in "--dim 1024" "--workload hek293" "--k 16" "--tol ppm:20 --workload hek293"; do for lib in build_ab/libstartsort.so ""; do
  echo "lib=${lib:-sum-order} $args"
  HOMS_B200_LIB=${lib:+$PWD/$lib} timeout 900 python bench.py $args --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "$show"
done; done ) > $O/r2_s24_ab_order.log 2>&1
cat $O/r2_s24_ab_order.log
