# GPU batch 7: A/B of work-item sizing at small D (same box, interleaved)
O=gpurun_out
show='import json,sys
for l in sys.stdin:
    l=l.strip()
    if not l.startswith("{"): continue
    j=json.loads(l); r=j["roofline"]
    print(" ms", round(j["ms_per_step"],3), "kernel", round(r["kernel_ms_per_launch"],3), "frac", round(r["frac"],3), "clk", j["clocks"]["sm_mhz"], j["clocks"]["reasons"])'
( for rep in 1 2; do for D in 1024 2048 4096; do for cfg in "0 0" "400 8" "200 16" "100 32" "64 64"; do
  set -- $cfg
  echo "rep=$rep dim=$D items_per_sm=$1 max_strip=$2 (0 = built-in)"
  if [ "$1" = "0" ]; then timeout 600 python bench.py --dim $D --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "$show"
  else HOMS_B200_TC_ITEMS_PER_SM=$1 HOMS_B200_TC_MAX_STRIP=$2 timeout 600 python bench.py --dim $D --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "$show"; fi
done; done; done ) > $O/r2_s07_item_sizing.log 2>&1
cat $O/r2_s07_item_sizing.log
