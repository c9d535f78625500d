# engine builds (LIBS) x configs (CFGS): DMMA chord launch time and fraction, 2 rounds
for i in 1 2; do
  for cfg in ${CFGS:-5 3}; do
    for lib in ${LIBS}; do
      MHAR_LIB=$lib timeout 300 python bench.py --config $cfg --no-i8 --no-fp32 --no-cpu --e2e-steps 1 --steps 10 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read().splitlines()[-1]);print('cfg $cfg $lib', round(d['roofline']['avg_launch_ms'],4), round(d['roofline']['frac'],4))"
    done
  done
done
