# GPU batch 30: stress of the CTA-pair hand-offs with one-row-tile work items
O=gpurun_out
HOMS_B200_TC_MAX_STRIP=1 HOMS_B200_TC_ITEMS_PER_SM=100000 timeout 1500 python tools/stress_pair.py --runs 300 > $O/r2_s30_stress_pair.log 2>&1; echo "rc=$?" >> $O/r2_s30_stress_pair.log
timeout 900 python tools/stress_pair.py --runs 200 --dims 4096 >> $O/r2_s30_stress_pair.log 2>&1; echo "rc=$?" >> $O/r2_s30_stress_pair.log
cat $O/r2_s30_stress_pair.log | tail -12
