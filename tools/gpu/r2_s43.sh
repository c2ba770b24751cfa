# GPU batch 43: B-tile evict_first hint under the pair kernel on the multi-group workloads
O=gpurun_out
show='import json,sys
for l in sys.stdin:
    l=l.strip()
    if not l.startswith("{"): continue
    j=json.loads(l); r=j["roofline"]
    print(" ms", round(j["ms_per_step"],4), "kernel", round(r["kernel_ms_per_launch"],4), "clk", j["clocks"]["sm_mhz"])'
for rep in 1 2; do for args in "--workload hek293" "--dim 16384" "--dim 2048" "--dim 1024"; do for h in 0 2; do echo "hints=$h $args rep=$rep"; HOMS_B200_TC_L2_HINTS=$h timeout 900 python bench.py $args --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "$show"; done; done; done
for h in 0 2; do
  HOMS_B200_TC_L2_HINTS=$h ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum --clock-control none -k regex:tc_search_kernel -s 3 -c 1 --csv --log-file $O/r2_s43_hek_hints$h.csv \
    python bench.py --workload hek293 --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
  echo "hek293 hints=$h"; grep "dram__bytes_read\|gpu__time" $O/r2_s43_hek_hints$h.csv | awk -F'","' '{print $(NF-2), $(NF-1), $NF}'
done
