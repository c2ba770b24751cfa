# GPU batch 3: measured L2 gather ceiling; L2 eviction hints x A-group budget on the search kernel (timing + DRAM bytes)
O=gpurun_out
tools/l2_gather_bench > $O/r2_s03_l2_gather.txt 2>&1
show='import json,sys
for l in sys.stdin:
    l=l.strip()
    if not l.startswith("{"): continue
    j=json.loads(l); r=j["roofline"]
    print(" ms", round(j["ms_per_step"],3), "kernel", round(r["kernel_ms_per_launch"],3), "frac", round(r["frac"],3), "clk", j["clocks"]["sm_mhz"], j["clocks"]["reasons"], "e2e", round(j["e2e"]["value"]))'
for rep in 1 2; do
for H in 0 1 2 3; do for GMB in 32 64; do
  echo "hints=$H group_mb=$GMB rep=$rep"
  HOMS_B200_TC_L2_HINTS=$H HOMS_B200_TC_GROUP_MB=$GMB timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "$show"
done; done; done > $O/r2_s03_hints_sweep.log 2>&1
M=dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,gpu__time_duration.sum,sm__pipe_tensor_subpipe_utcomma_cycles_active.avg.pct_of_peak_sustained_elapsed,l1tex__m_xbar2l1tex_read_bytes.sum
for H in 0 3; do for GMB in 32 64; do
  HOMS_B200_TC_L2_HINTS=$H HOMS_B200_TC_GROUP_MB=$GMB timeout 900 ncu --metrics $M --clock-control none -k regex:tc_search_kernel -c 2 --csv \
    --log-file $O/r2_s03_ncu_dram_h${H}_g${GMB}.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
done; done
tail -20 $O/r2_s03_hints_sweep.log
