# GPU batch 26: where does D = 1024 lose?  ncu source capture of the single-CTA kernel at D = 1024
O=gpurun_out
ncu --set full --clock-control none --import-source on -k regex:tc_search_kernel -s 3 -c 1 -f -o $O/r2_s26_search_d1024 \
  python bench.py --dim 1024 --steps 1 --warmup 3 --no-cpu-baseline > $O/r2_s26_ncu.log 2>&1
ncu -i $O/r2_s26_search_d1024.ncu-rep --page raw --csv > $O/r2_s26_raw.csv 2>/dev/null
ncu -i $O/r2_s26_search_d1024.ncu-rep --page source --csv > $O/r2_s26_source.csv 2>/dev/null
python tools/ncu_summary.py $O/r2_s26_raw.csv | head -24
