# chord3 TMEM hand-off barriers per twin pair (default build) vs one 8-arrival
# barrier per buffer (tools/build_ab.sh pair0 "-DMHAR_C3_PAIRBAR=0"), configs 3/4/5
for i in 1 2; do
  for cfg in ${CFGS:-3 4 5}; do
    for lib in paper_2104_07097_b200/lib/libmhar_b200.so tools/ab_pair0.so; do
      MHAR_LIB=$lib timeout 300 python bench.py --config $cfg --no-i8 --no-fp32 --no-cpu --e2e-steps 1 --steps 10 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read().splitlines()[-1]);print('cfg $cfg $lib', round(d['roofline']['avg_launch_ms'],4), round(d['roofline']['frac'],4), round(d['value']), d['checks']['all_inside_eps_feas'])"
    done
  done
done
