# GPU batch 36: planner knobs under the pair kernel (config 2 and config-3 prefix)
O=gpurun_out
show='import json,sys
for l in sys.stdin:
    l=l.strip()
    if not l.startswith("{"): continue
    j=json.loads(l); r=j["roofline"]
    print(" ms", round(j["ms_per_step"],4), "kernel", round(r["kernel_ms_per_launch"],4), "clk", j["clocks"]["sm_mhz"], "frac", round(r.get("frac") or 0,4))'
( for rep in 1 2; do
echo "default rep=$rep"; timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "$show"
for v in 200 800; do echo "items_per_sm=$v rep=$rep"; HOMS_B200_TC_ITEMS_PER_SM=$v timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "$show"; done
for v in 4 16; do echo "max_strip=$v rep=$rep"; HOMS_B200_TC_MAX_STRIP=$v timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "$show"; done
for v in 32 48; do echo "group_mb=$v rep=$rep"; HOMS_B200_TC_GROUP_MB=$v timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "$show"; done
done
echo "hek293 default"; timeout 900 python bench.py --workload hek293 --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "$show"
for v in 16 48 64; do echo "hek293 group_mb=$v"; HOMS_B200_TC_GROUP_MB=$v timeout 900 python bench.py --workload hek293 --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "$show"; done
for v in 200 800; do echo "hek293 items_per_sm=$v"; HOMS_B200_TC_ITEMS_PER_SM=$v timeout 900 python bench.py --workload hek293 --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "$show"; done
) > $O/r2_s36_knobs_pair.log 2>&1
cat $O/r2_s36_knobs_pair.log
