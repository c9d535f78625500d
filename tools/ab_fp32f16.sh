# fp32 variant (fp16 form) A/B of engine builds: avg tc32 launch ms and clock
libs=${LIBS:-"paper_2104_07097_b200/lib/libmhar_b200.so"}
for i in 1 2 3; do
  for lib in $libs; do
    MHAR_LIB=$lib timeout 120 python bench.py --precision 32 --no-i8 --no-fp32 --no-cpu --e2e-steps 1 --steps 20 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read().splitlines()[-1]);print('$lib', round(d['roofline']['avg_launch_ms'],3), round(d['value']))"
  done
done
