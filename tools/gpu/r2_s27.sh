# GPU batch 27: resident query chunks for D <= 1024 (single CTAs): suite, interleaved A/B, item length
O=gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q --deselect tests/test_whole_config_gpu.py > $O/r2_s27_tests.log 2>&1; echo "rc=$?" >> $O/r2_s27_tests.log
tail -4 $O/r2_s27_tests.log
show='import json,sys
for l in sys.stdin:
    l=l.strip()
    if not l.startswith("{"): continue
    j=json.loads(l); r=j["roofline"]
    print(" ms", round(j["ms_per_step"],4), "kernel", round(r["kernel_ms_per_launch"],4), "clk", j["clocks"]["sm_mhz"], "frac", round(r.get("frac") or 0,4), "e2e", round(j["e2e"]["value"]))'
( for rep in 1 2; do for ares in 0 1; do
  echo "ares=$ares D=1024 rep=$rep"; HOMS_B200_TC_ARES=$ares timeout 600 python bench.py --dim 1024 --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "$show"
done; done
for ares in 0 1; do echo "ares=$ares hek293 D=1024"; HOMS_B200_TC_ARES=$ares timeout 900 python bench.py --workload hek293 --dim 1024 --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "$show"; done
for ares in 0 1; do echo "ares=$ares D=512"; HOMS_B200_TC_ARES=$ares timeout 900 python bench.py --dim 512 --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "$show"; done
for ms in 16 64 128; do echo "ares=1 D=1024 max_strip=$ms"; HOMS_B200_TC_MAX_STRIP=$ms timeout 600 python bench.py --dim 1024 --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "$show"; done
for ips in 50 200; do echo "ares=1 D=1024 items_per_sm=$ips"; HOMS_B200_TC_ITEMS_PER_SM=$ips timeout 600 python bench.py --dim 1024 --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "$show"; done
echo "pair=1 D=1024"; HOMS_B200_TC_PAIR=1 timeout 600 python bench.py --dim 1024 --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "$show"
) > $O/r2_s27_ab_ares.log 2>&1
cat $O/r2_s27_ab_ares.log
