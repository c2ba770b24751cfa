# GPU batch 33: ncu source capture at D = 1024 with resident query chunks
O=gpurun_out
ncu --set full --clock-control none --import-source on -k regex:tc_search_kernel -s 3 -c 1 -f -o $O/r2_s33_d1024 \
  python bench.py --dim 1024 --steps 1 --warmup 3 --no-cpu-baseline > $O/r2_s33_ncu.log 2>&1
ncu -i $O/r2_s33_d1024.ncu-rep --page raw --csv > $O/r2_s33_raw.csv 2>/dev/null
ncu -i $O/r2_s33_d1024.ncu-rep --page source --csv > $O/r2_s33_source.csv 2>/dev/null
python tools/ncu_summary.py $O/r2_s33_raw.csv | head -22
