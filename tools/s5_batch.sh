#!/bin/bash
# one gpurun batch: encode ncu capture, sanitizer pass, bench lines (development aid)
O=gpurun_out
ncu --set full --clock-control none --import-source on -k regex:encode_kernel -c 1 -o $O/s5_encode_full -f \
  python bench.py --workload encode --steps 1 --warmup 3 --no-cpu-baseline --encode-spectra 250000 > $O/s5_ncu_encode.log 2>&1
timeout 900 compute-sanitizer --tool memcheck --error-exitcode 9 \
  python -m pytest tests/test_encode_gpu.py tests/test_fused_gpu.py -m gpu -x -q > $O/s5_sanitizer_encode.log 2>&1
echo "memcheck encode rc=$?" >> $O/s5_sanitizer_encode.log
timeout 1200 compute-sanitizer --tool memcheck --error-exitcode 9 \
  python -m pytest tests/test_search_gpu.py -m gpu -x -q -k "golden or known_answers or topk" > $O/s5_sanitizer_search.log 2>&1
echo "memcheck search rc=$?" >> $O/s5_sanitizer_search.log
python bench.py --workload encode --steps 3 --warmup 3 > $O/s5_bench_encode.json 2> $O/s5_bench_encode.err
python bench.py --steps 5 --warmup 3 > $O/s5_bench_default.json 2> $O/s5_bench_default.err
python bench.py --steps 5 --warmup 3 --k 5 --no-cpu-baseline > $O/s5_bench_k5.json 2> $O/s5_bench_k5.err
python bench.py --steps 5 --warmup 3 --k 16 --no-cpu-baseline > $O/s5_bench_k16.json 2> $O/s5_bench_k16.err
