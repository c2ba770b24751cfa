# GPU batch 22: pair threshold (D = 2048 / 4096), ncu captures of the default kernels, launch list, sanitizers
O=gpurun_out
show='import json,sys
for l in sys.stdin:
    l=l.strip()
    if not l.startswith("{"): continue
    j=json.loads(l); r=j["roofline"]
    print(" ms", round(j["ms_per_step"],4), "kernel", round(r["kernel_ms_per_launch"],4), "clk", j["clocks"]["sm_mhz"], "frac", round(r.get("frac") or 0,4), "probe", round(r["peak"]), "e2e", round(j["e2e"]["value"]))'
( for rep in 1 2; do for args in "--dim 2048" "--dim 4096" "--workload hek293 --dim 2048"; do for pair in 0 1; do
  echo "pair=$pair $args rep=$rep"
  HOMS_B200_TC_PAIR=$pair timeout 900 python bench.py $args --steps 8 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "$show"
done; done; done ) > $O/r2_s22_ab_pair_threshold.log 2>&1
cat $O/r2_s22_ab_pair_threshold.log
ncu --set full --clock-control none --import-source on -k regex:tc_search_kernel -s 3 -c 1 -f -o $O/r2_s22_search_top1 \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $O/r2_s22_ncu_top1.log 2>&1
ncu -i $O/r2_s22_search_top1.ncu-rep --page raw --csv > $O/r2_s22_search_top1_raw.csv 2>/dev/null
python tools/ncu_summary.py $O/r2_s22_search_top1_raw.csv > $O/r2_s22_search_top1_ncu.csv
ncu --set full --clock-control none --import-source on -k regex:tc_search_kernel -s 3 -c 1 -f -o $O/r2_s22_search_k16 \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline --k 16 > $O/r2_s22_ncu_k16.log 2>&1
ncu -i $O/r2_s22_search_k16.ncu-rep --page raw --csv > $O/r2_s22_search_k16_raw.csv 2>/dev/null
python tools/ncu_summary.py $O/r2_s22_search_k16_raw.csv > $O/r2_s22_search_k16_ncu.csv
ncu --set full --clock-control none -k regex:encode_kernel -s 2 -c 1 -f -o $O/r2_s22_encode \
  python bench.py --workload encode --encode-spectra 1000000 --steps 1 --warmup 1 --no-cpu-baseline > $O/r2_s22_ncu_encode.log 2>&1
ncu -i $O/r2_s22_encode.ncu-rep --page raw --csv > $O/r2_s22_encode_raw.csv 2>/dev/null
python tools/ncu_summary.py $O/r2_s22_encode_raw.csv > $O/r2_s22_encode_ncu.csv
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/r2_s22_launches_default.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/r2_s22_launches.log 2>&1
head -12 $O/r2_s22_search_top1_ncu.csv
timeout 1800 compute-sanitizer --tool memcheck --error-exitcode 9 \
  python -m pytest tests/test_search_gpu.py tests/test_multi_device_gpu.py tests/test_pipeline_gpu.py tests/test_mgf_gpu.py -m gpu -x -q \
  -k "golden or known_answers or topk_vs_port or group_search or query_file or engine_selection or kernel_forms or index_order or mgf_golden or topk_modes" > $O/r2_s22_memcheck.log 2>&1
echo "memcheck rc=$?" >> $O/r2_s22_memcheck.log
timeout 1500 compute-sanitizer --tool racecheck --error-exitcode 9 \
  python -m pytest tests/test_search_gpu.py -m gpu -x -q -k "golden or kernel_forms or index_order" > $O/r2_s22_racecheck.log 2>&1
echo "racecheck rc=$?" >> $O/r2_s22_racecheck.log
timeout 900 compute-sanitizer --tool memcheck --error-exitcode 9 \
  python -m pytest tests/test_encode_gpu.py tests/test_fused_gpu.py tests/test_cache.py -m gpu -x -q > $O/r2_s22_memcheck_encode.log 2>&1
echo "memcheck encode/fused/cache rc=$?" >> $O/r2_s22_memcheck_encode.log
tail -3 $O/r2_s22_memcheck.log; tail -3 $O/r2_s22_racecheck.log; tail -3 $O/r2_s22_memcheck_encode.log
