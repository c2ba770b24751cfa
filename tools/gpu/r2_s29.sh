# GPU batch 29: shorter radix chunks at query counts, four records in flight in the reduce: suite + launch list + shard projection
O=gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q --deselect tests/test_whole_config_gpu.py > $O/r2_s29_tests.log 2>&1; echo "rc=$?" >> $O/r2_s29_tests.log
tail -4 $O/r2_s29_tests.log
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/r2_s29_launches_default.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/r2_s29_launches.log 2>&1
timeout 1500 python tools/shard_sim.py --shards 1,2,4,8 --steps 5 > $O/r2_s29_shard_sim.jsonl 2> $O/r2_s29_shard_sim.err
head -4 $O/r2_s29_shard_sim.jsonl | cut -c 1-330
show='import json,sys
for l in sys.stdin:
    l=l.strip()
    if not l.startswith("{"): continue
    j=json.loads(l); r=j["roofline"]
    print(" ms", round(j["ms_per_step"],4), "kernel", round(r["kernel_ms_per_launch"],4), "clk", j["clocks"]["sm_mhz"], "e2e", round(j["e2e"]["value"]))'
for args in "" "--workload hek293 --tol ppm:100" "--tol ppm:20"; do echo "bench $args"; timeout 900 python bench.py $args --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "$show"; done
