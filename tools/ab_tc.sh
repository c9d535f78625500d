# A/B of the fp32 variant's kernel: env settings x direction forms, 2 rounds
for i in 1 2; do
  for dir in split rounded; do
    for envs in ${ENVS:-"MHAR_TC_TMA=1" "MHAR_TC_TMA=0"}; do
      env $envs timeout 300 python bench.py --precision 32 --fp32-direction $dir --no-i8 --no-fp32 --no-cpu --e2e-steps 1 --steps 10 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read().splitlines()[-1]);print('$dir $envs', round(d['roofline']['avg_launch_ms'],4), round(d['roofline']['achieved'],1), d['clocks']['sm_mhz'], round(d['value']))"
    done
  done
done
