for i in 1 2; do
  for cfg in ${CFGS:-5 3 4}; do
    for v in "tools/ab_base.so 0" "tools/ab_c3int.so 0" "tools/ab_c3.so 1" "tools/ab_c3int.so 1"; do
      set -- $v
      MHAR_LIB=$1 MHAR_CHORD3=$2 timeout 300 python bench.py --config $cfg --no-i8 --no-fp32 --no-cpu --e2e-steps 1 --steps 10 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read().splitlines()[-1]);print('cfg $cfg $1 chord3=$2', round(d['roofline']['avg_launch_ms'],4), round(d['roofline']['frac'],4))"
    done
  done
done
