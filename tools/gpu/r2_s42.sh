# GPU batch 42: L2 eviction hints under the pair kernel: DRAM bytes (ncu, two metrics) and live timings
O=gpurun_out
for h in 0 2 3; do
  HOMS_B200_TC_L2_HINTS=$h ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum --clock-control none -k regex:tc_search_kernel -s 3 -c 1 --csv --log-file $O/r2_s42_hints$h.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
  echo "hints=$h"; grep "dram__bytes_read\|gpu__time" $O/r2_s42_hints$h.csv | awk -F'","' '{print $(NF-2), $(NF-1), $NF}'
done
for g in 32 48; do
  HOMS_B200_TC_GROUP_MB=$g ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum --clock-control none -k regex:tc_search_kernel -s 3 -c 1 --csv --log-file $O/r2_s42_group$g.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
  echo "group_mb=$g"; grep "dram__bytes_read\|gpu__time" $O/r2_s42_group$g.csv | awk -F'","' '{print $(NF-2), $(NF-1), $NF}'
done
show='import json,sys
for l in sys.stdin:
    l=l.strip()
    if not l.startswith("{"): continue
    j=json.loads(l); r=j["roofline"]
    print(" ms", round(j["ms_per_step"],4), "kernel", round(r["kernel_ms_per_launch"],4), "clk", j["clocks"]["sm_mhz"])'
for rep in 1 2; do for h in 0 2; do echo "live hints=$h rep=$rep"; HOMS_B200_TC_L2_HINTS=$h timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "$show"; done; done
