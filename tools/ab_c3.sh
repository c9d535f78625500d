# chord3 (warp-specialised through TMEM) vs chord2 (MHAR_CHORD3=0) on the DMMA incremental path
for i in 1 2; do
  for cfg in ${CFGS:-5 3 4}; do
    for v in 1 0; do
      MHAR_CHORD3=$v timeout 300 python bench.py --config $cfg --no-i8 --no-fp32 --no-cpu --e2e-steps 1 --steps 10 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read().splitlines()[-1]);print('cfg $cfg chord3=$v', round(d['roofline']['avg_launch_ms'],4), round(d['roofline']['frac'],4), round(d['value']), d['checks']['all_inside_eps_feas'])"
    done
  done
done
