# GPU batch 25: final evidence of round 2 -- every bench line, ncu captures, launch list (tests and sanitizers: r2_s23/24)
O=gpurun_out
python bench.py --steps 20 --warmup 5 > $O/final_bench_default.json 2> $O/final_bench_default.err
python bench.py --impl reference --steps 5 --warmup 1 > $O/final_bench_reference.json 2> $O/final_bench_reference.err
for k in 5 16 17 32 33 64; do timeout 900 python bench.py --k $k --steps 10 --warmup 3 > $O/final_bench_top$k.json 2> $O/final_bench_top$k.err; done
timeout 900 python bench.py --tol ppm:20 --steps 50 --warmup 5 > $O/final_bench_ppm20.json 2> $O/final_bench_ppm20.err
timeout 1800 python bench.py --workload hek293 --steps 5 --warmup 3 > $O/final_bench_hek293_prefix.json 2> $O/final_bench_hek293_prefix.err
timeout 3000 python bench.py --workload hek293_full --steps 3 --warmup 3 > $O/final_bench_hek293_full_1M.json 2> $O/final_bench_hek293_full_1M.err
timeout 1800 python bench.py --workload encode --steps 3 --warmup 3 > $O/final_bench_encode_config4_10M.json 2> $O/final_bench_encode_config4_10M.err
timeout 1800 python bench.py --workload encode --encode-max-peaks 50 --steps 3 --warmup 3 > $O/final_bench_encode_config4_10M_top50.json 2> $O/final_bench_encode_top50.err
timeout 1800 python bench.py --workload pipeline --steps 5 --warmup 3 > $O/final_bench_pipeline_query_file.json 2> $O/final_bench_pipeline.err
timeout 1800 python bench.py --workload mgf --steps 5 --warmup 3 > $O/final_bench_mgf_parse.json 2> $O/final_bench_mgf.err
timeout 3000 python tools/config5_sweep.py > $O/final_config5_sweep_1gpu.jsonl 2> $O/final_config5_sweep.err
ncu --set full --clock-control none --import-source on -k regex:tc_search_kernel -s 3 -c 1 -f -o $O/final_search_top1 \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $O/final_ncu_top1.log 2>&1
ncu -i $O/final_search_top1.ncu-rep --page raw --csv > $O/final_search_top1_raw.csv 2>/dev/null
python tools/ncu_summary.py $O/final_search_top1_raw.csv > $O/final_search_top1_ncu.csv
ncu --set full --clock-control none --import-source on -k "regex:tc_search_kernel<\(int\)0" -s 3 -c 1 -f -o $O/final_search_k16 \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline --k 16 > $O/final_ncu_k16.log 2>&1
ncu -i $O/final_search_k16.ncu-rep --page raw --csv > $O/final_search_k16_raw.csv 2>/dev/null
python tools/ncu_summary.py $O/final_search_k16_raw.csv > $O/final_search_k16_ncu.csv
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/final_launches_default.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/final_launches.log 2>&1
for f in default reference top5 top16 top17 top32 top33 top64 ppm20 hek293_prefix hek293_full_1M encode_config4_10M encode_config4_10M_top50 pipeline_query_file mgf_parse; do
  python - "$O/final_bench_$f.json" <<'E'
import json,sys
try:
    j=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    print(sys.argv[1].split("final_bench_")[1], "value", round(j.get("value") or 0,1), j.get("unit"), "ms", round(j.get("ms_per_step") or 0,3), "e2e", j.get("e2e") and round(j["e2e"]["value"],1), "frac", j.get("roofline") and j["roofline"].get("frac"), "cpu", j.get("cpu_baseline") and j["cpu_baseline"].get("value"))
except Exception as e: print(sys.argv[1], "FAILED", e)
E
done
head -8 $O/final_search_top1_ncu.csv; head -8 $O/final_search_k16_ncu.csv
