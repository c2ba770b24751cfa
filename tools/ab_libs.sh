# development A/B: default build vs experimental builds of the library (HOMS_B200_LIB)
for lib in "" build/libexp_224_5.so build/libexp_208_5.so ""; do
  echo "lib=${lib:-default}"
  HOMS_B200_LIB=${lib:+$PWD/$lib} python bench.py --no-cpu-baseline --steps 8 2>/dev/null | python -c "import json,sys; j=json.loads(sys.stdin.read()); r=j['roofline']; print(' ms', round(j['ms_per_step'],3), 'q/s', round(j['value']), 'kernel_ms', round(r['kernel_ms_per_launch'],3), 'frac', round(r['frac'],3), 'clk', j['clocks']['sm_mhz'])"
done
