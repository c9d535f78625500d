# A/B of an environment knob on the DMMA headline (config 5)
for i in 1 2; do
  for v in ${VALS:-2 4 8 16}; do
    env ${KNOB:-MHAR_GROUP_M}=$v timeout 200 python bench.py --no-i8 --no-fp32 --no-cpu --e2e-steps 1 --steps 10 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read().splitlines()[-1]);print('${KNOB:-MHAR_GROUP_M}=$v', round(d['roofline']['avg_launch_ms'],3), round(d['roofline']['frac'],4))"
  done
done
