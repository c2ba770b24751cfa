#!/bin/bash
# compute-sanitizer passes over the search engines (development aid)
O=gpurun_out
timeout 1500 compute-sanitizer --tool memcheck --error-exitcode 9 \
  python -m pytest tests/test_search_gpu.py -m gpu -x -q -k "golden or known_answers or topk_vs_port or sharded or engine_selection" > $O/sanitize_memcheck_search.log 2>&1
echo "memcheck search rc=$?" >> $O/sanitize_memcheck_search.log
timeout 1500 compute-sanitizer --tool racecheck --error-exitcode 9 \
  python -m pytest tests/test_search_gpu.py -m gpu -x -q -k "golden or topk_vs_port" > $O/sanitize_racecheck_search.log 2>&1
echo "racecheck search rc=$?" >> $O/sanitize_racecheck_search.log
timeout 900 compute-sanitizer --tool memcheck --error-exitcode 9 \
  python -m pytest tests/test_encode_gpu.py tests/test_fused_gpu.py tests/test_cache.py -m gpu -x -q > $O/sanitize_memcheck_encode.log 2>&1
echo "memcheck encode/fused/cache rc=$?" >> $O/sanitize_memcheck_encode.log
