# GPU batch 28: shard projection with the round-2 kernels; bench.py --gpus 2 functional check (ranks share the GPU); group context bench
O=gpurun_out
timeout 1500 python tools/shard_sim.py --shards 1,2,4,8 --steps 5 > $O/r2_s28_shard_sim.jsonl 2> $O/r2_s28_shard_sim.err
cat $O/r2_s28_shard_sim.jsonl | tail -6
timeout 1500 python bench.py --gpus 2 --steps 3 --warmup 3 --no-cpu-baseline > $O/r2_s28_bench_gpus2.json 2> $O/r2_s28_bench_gpus2.err
tail -c 1500 $O/r2_s28_bench_gpus2.json; tail -3 $O/r2_s28_bench_gpus2.err
