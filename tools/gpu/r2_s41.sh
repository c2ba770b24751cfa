# GPU batch 41: ncu capture of the collect-mode search kernel (k = 16)
O=gpurun_out
ncu --set full --clock-control none --import-source on -k regex:tc_search_kernel -s 6 -c 1 -f -o $O/r2_s41_search_k16 \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline --k 16 > $O/r2_s41_ncu_k16.log 2>&1
ncu -i $O/r2_s41_search_k16.ncu-rep --page raw --csv > $O/r2_s41_search_k16_raw.csv 2>/dev/null
python tools/ncu_summary.py $O/r2_s41_search_k16_raw.csv | head -24
