libs=${LIBS:-"tools/ab_lag1.so tools/ab_lag2.so"}
for i in 1 2; do
  for lib in $libs; do
    MHAR_LIB=$lib timeout 200 python bench.py --no-i8 --no-fp32 --no-cpu --e2e-steps 1 --steps 10 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read().splitlines()[-1]);print('$lib', round(d['roofline']['avg_launch_ms'],3), round(d['roofline']['frac'],4), d['clocks']['sm_mhz'])"
  done
done
