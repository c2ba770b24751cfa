# GPU batch 40: sanitizers on the final build
O=gpurun_out
timeout 1800 compute-sanitizer --tool memcheck --error-exitcode 9 \
  python -m pytest tests/test_search_gpu.py tests/test_multi_device_gpu.py tests/test_pipeline_gpu.py tests/test_mgf_gpu.py -m gpu -x -q \
  -k "golden or known_answers or topk_vs_port or group_search or query_file or engine_selection or kernel_forms or index_order or mgf_golden or topk_modes or planning_batches" > $O/r2_s40_memcheck.log 2>&1
echo "memcheck rc=$?" >> $O/r2_s40_memcheck.log
timeout 1500 compute-sanitizer --tool racecheck --error-exitcode 9 \
  python -m pytest tests/test_search_gpu.py -m gpu -x -q -k "golden or kernel_forms or index_order" > $O/r2_s40_racecheck.log 2>&1
echo "racecheck rc=$?" >> $O/r2_s40_racecheck.log
timeout 900 compute-sanitizer --tool memcheck --error-exitcode 9 \
  python -m pytest tests/test_encode_gpu.py tests/test_fused_gpu.py tests/test_cache.py -m gpu -x -q > $O/r2_s40_memcheck_encode.log 2>&1
echo "memcheck encode/fused/cache rc=$?" >> $O/r2_s40_memcheck_encode.log
timeout 900 compute-sanitizer --tool initcheck --error-exitcode 9 \
  python -m pytest tests/test_search_gpu.py -m gpu -x -q -k "golden or kernel_forms or index_order" > $O/r2_s40_initcheck.log 2>&1
echo "initcheck rc=$?" >> $O/r2_s40_initcheck.log
tail -3 $O/r2_s40_memcheck.log; grep "Race reported\|and " $O/r2_s40_racecheck.log | sed 's/+0x[0-9a-f]*//g' | sed 's/<(int)[0-9]*, /<KM, /' | sort | uniq -c | sort -rn | head -12; tail -3 $O/r2_s40_racecheck.log; tail -3 $O/r2_s40_memcheck_encode.log; tail -4 $O/r2_s40_initcheck.log
