# fp32 variant A/B: engine builds (LIBS) x configs (CFGS) x direction forms
for i in 1 2; do
  for cfg in ${CFGS:-3 4 5}; do
    for dir in split rounded; do
      for lib in ${LIBS}; do
        MHAR_LIB=$lib timeout 300 python bench.py --config $cfg --precision 32 --fp32-direction $dir --no-i8 --no-cpu --e2e-steps 1 --steps 10 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read().splitlines()[-1]);print('cfg $cfg $dir $lib', round(d['value']), round(d['roofline']['avg_launch_ms'],4), round(d['roofline']['frac'],4))"
      done
    done
  done
done
