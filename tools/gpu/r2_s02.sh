set -x
O=gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q --durations=15 > $O/r2_s02_tests.log 2>&1; echo "tests rc=$?" >> $O/r2_s02_tests.log
for k in 16 17 32 33 64; do
  timeout 600 python bench.py --steps 5 --warmup 3 --k $k --no-cpu-baseline > $O/r2_s02_bench_k$k.json 2> $O/r2_s02_bench_k$k.err
done
timeout 900 python bench.py --workload encode --steps 3 --warmup 3 > $O/r2_s02_bench_encode.json 2> $O/r2_s02_bench_encode.err
timeout 900 python bench.py --workload pipeline --steps 5 --warmup 3 > $O/r2_s02_bench_pipeline.json 2> $O/r2_s02_bench_pipeline.err
timeout 900 python bench.py --gpus 2 --steps 3 --warmup 3 > $O/r2_s02_bench_gpus2.json 2> $O/r2_s02_bench_gpus2.err
tail -5 $O/r2_s02_tests.log
