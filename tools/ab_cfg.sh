# A/B of engine builds on BASELINE configs 3 and 4 (DMMA headline engine)
libs=${LIBS:-"tools/ab_p0.so tools/ab_p1.so"}
for cfg in ${CFGS:-3 4}; do
for i in 1 2; do
  for lib in $libs; do
    MHAR_LIB=$lib timeout 200 python bench.py --config $cfg --no-i8 --no-fp32 --no-cpu --e2e-steps 1 --steps 10 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read().splitlines()[-1]);print('cfg $cfg', '$lib', round(d['roofline']['avg_launch_ms'],3), round(d['roofline']['frac'],4))"
  done
done
done
