# GPU batch 19: interleaved A/B on one box: single-thread roles behind `lane == 0` (round 1) vs elect.sync
O=gpurun_out
show='import json,sys
for l in sys.stdin:
    l=l.strip()
    if not l.startswith("{"): continue
    j=json.loads(l); r=j["roofline"]
    print(" ms", round(j["ms_per_step"],4), "kernel", round(r["kernel_ms_per_launch"],4), "clk", j["clocks"]["sm_mhz"], "frac", round(r.get("frac") or 0,4), "probe", round(r["peak"]), "e2e", round(j["e2e"]["value"]))'
( for rep in 1 2 3; do for lib in build_ab/libnoelect.so ""; do
  echo "lib=${lib:-elect} rep=$rep"
  HOMS_B200_LIB=${lib:+$PWD/$lib} timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "$show"
done; done
for args in "--dim 1024" "--dim 16384" "--workload hek293" "--k 16"; do for lib in build_ab/libnoelect.so ""; do
  echo "lib=${lib:-elect} $args"
  HOMS_B200_LIB=${lib:+$PWD/$lib} timeout 900 python bench.py $args --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "$show"
done; done ) > $O/r2_s19_ab_elect.log 2>&1
cat $O/r2_s19_ab_elect.log
( echo "encode max_peaks=50 of 150 raw peaks"; timeout 900 python bench.py --workload encode --encode-spectra 2000000 --encode-max-peaks 50 --steps 3 --warmup 3 2>&1 | tail -1 | python -c "
import json,sys
j=json.loads(sys.stdin.read()); r=j['roofline']; print(j['value'], j['ms_per_step'], r.get('preprocess_share_of_step'), j['cpu_baseline'].get('parity_with_gpu_on_sample'))"
) > $O/r2_s19_encode_topn.log 2>&1
cat $O/r2_s19_encode_topn.log
