# GPU batch 17: ncu full capture with source of the top-1 search kernel (where do the 7 % of idle tensor cycles go?),
# launch list of the default step
O=gpurun_out
ncu --set full --clock-control none --import-source on -k regex:tc_search_kernel -s 3 -c 1 -f -o $O/r2_s17_search_top1 \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $O/r2_s17_ncu_top1.log 2>&1
ncu -i $O/r2_s17_search_top1.ncu-rep --page raw --csv > $O/r2_s17_search_top1_raw.csv 2>/dev/null
ncu -i $O/r2_s17_search_top1.ncu-rep --page source --csv > $O/r2_s17_search_top1_source.csv 2>/dev/null
ls -la $O/r2_s17_search_top1*
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/r2_s17_launches_default.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline > $O/r2_s17_launches.log 2>&1
python tools/ncu_summary.py $O/r2_s17_search_top1_raw.csv | head -60
