# GPU batch 20: CTA pairs again now that the issue threads are lean (interleaved A/B), ncu source capture of the new kernel
O=gpurun_out
show='import json,sys
for l in sys.stdin:
    l=l.strip()
    if not l.startswith("{"): continue
    j=json.loads(l); r=j["roofline"]
    print(" ms", round(j["ms_per_step"],4), "kernel", round(r["kernel_ms_per_launch"],4), "clk", j["clocks"]["sm_mhz"], "frac", round(r.get("frac") or 0,4), "probe", round(r["peak"]), "e2e", round(j["e2e"]["value"]))'
HOMS_B200_LIB=$PWD/build_ab/libpair.so HOMS_B200_TC_PAIR=1 timeout 900 python -m pytest tests/test_search_gpu.py -m gpu -x -q -k "tensor or auto or topk or planning or tight" > $O/r2_s20_tests_pair.log 2>&1; echo "rc=$?" >> $O/r2_s20_tests_pair.log
tail -3 $O/r2_s20_tests_pair.log
( for rep in 1 2 3; do for pair in 0 1; do
  echo "pair=$pair rep=$rep"
  HOMS_B200_LIB=$PWD/build_ab/libpair.so HOMS_B200_TC_PAIR=$pair timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "$show"
done; done
for args in "--dim 1024" "--dim 16384" "--workload hek293"; do for pair in 0 1; do
  echo "pair=$pair $args"
  HOMS_B200_LIB=$PWD/build_ab/libpair.so HOMS_B200_TC_PAIR=$pair timeout 900 python bench.py $args --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "$show"
done; done ) > $O/r2_s20_ab_pair_elect.log 2>&1
cat $O/r2_s20_ab_pair_elect.log
ncu --set full --clock-control none --import-source on -k regex:tc_search_kernel -s 3 -c 1 -f -o $O/r2_s20_search_top1 \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $O/r2_s20_ncu_top1.log 2>&1
ncu -i $O/r2_s20_search_top1.ncu-rep --page raw --csv > $O/r2_s20_search_top1_raw.csv 2>/dev/null
ncu -i $O/r2_s20_search_top1.ncu-rep --page source --csv > $O/r2_s20_search_top1_source.csv 2>/dev/null
python tools/ncu_summary.py $O/r2_s20_search_top1_raw.csv | head -24
