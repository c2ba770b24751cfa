# GPU batch 45: query-tile group size on the config-3 prefix with the eviction hints off
O=gpurun_out
show='import json,sys
for l in sys.stdin:
    l=l.strip()
    if not l.startswith("{"): continue
    j=json.loads(l); r=j["roofline"]
    print(" ms", round(j["ms_per_step"],4), "kernel", round(r["kernel_ms_per_launch"],4), "clk", j["clocks"]["sm_mhz"], "frac", round(r.get("frac") or 0,4))'
( for v in 32 16 24 48 64; do echo "hek293 group_mb=$v"; HOMS_B200_TC_GROUP_MB=$v timeout 900 python bench.py --workload hek293 --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "$show"; done
echo "hek293 default again"; timeout 900 python bench.py --workload hek293 --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "$show" ) > $O/r2_s45_group_hek.log 2>&1
cat $O/r2_s45_group_hek.log
