# GPU batch 5: pipelined encode kernel -- parity tests, A/B against the unpipelined build, ncu
O=gpurun_out
timeout 900 python -m pytest tests/test_encode_gpu.py tests/test_fused_gpu.py tests/test_pipeline_gpu.py -m gpu -x -q > $O/r2_s05_tests.log 2>&1; echo "rc=$?" >> $O/r2_s05_tests.log
for rep in 1 2; do
bash tools/ab_encode.sh $PWD/build/libenc_nopipe.so $PWD/paper_2211_16422_b200/libhoms_b200.so
done > $O/r2_s05_ab_encode.log 2>&1
for mp in 150 50; do
for lib in $PWD/build/libenc_nopipe.so $PWD/paper_2211_16422_b200/libhoms_b200.so; do
  echo "== max_peaks=$mp $lib"
  HOMS_B200_LIB=$lib python bench.py --workload encode --steps 3 --warmup 3 --no-cpu-baseline --encode-spectra 2000000 --encode-max-peaks $mp 2>/dev/null | python -c "
import json,sys
j=json.loads(sys.stdin.read()); r=j['roofline']
print('spectra/s %.4g  encode_kernel_ms %.3f  share %.3f  pre_share %.3f e2e %.4g  clk %s' % (j['value'], r['kernel_ms_per_launch'], r['kernel_share_of_step'], r['preprocess_share_of_step'], j['e2e']['value'], j['clocks']['sm_mhz']))"
done; done >> $O/r2_s05_ab_encode.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:encode_kernel -s 4 -c 1 -o $O/r2_s05_encode_full -f python bench.py --workload encode --steps 1 --warmup 3 --no-cpu-baseline --encode-spectra 1000000 > /dev/null 2>&1
ncu -i $O/r2_s05_encode_full.ncu-rep --page raw --csv > $O/r2_s05_encode_full_raw.csv 2>/dev/null
cat $O/r2_s05_tests.log | tail -3; cat $O/r2_s05_ab_encode.log
