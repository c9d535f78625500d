# int8 engine wait counters (MHAR_I8_PROFILE=1) for each library in $LIBS
libs=${LIBS:-"paper_2104_07097_b200/lib/libmhar_b200.so"}
for lib in $libs; do
  echo "== $lib"
  MHAR_I8_PROFILE=1 MHAR_LIB=$lib timeout 120 python bench.py --f64-engine int8 --no-i8 --no-fp32 --no-cpu --e2e-steps 1 --steps 10 2>&1 | grep "tcgen05 profile" | tail -2
done
