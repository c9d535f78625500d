# fp32-variant wait counters (MHAR_I8_PROFILE=1) for each form
for f in 1 0; do
  echo "== MHAR_TC_F16=$f"
  MHAR_TC_F16=$f MHAR_I8_PROFILE=1 timeout 120 python bench.py --precision 32 --no-i8 --no-fp32 --no-cpu --e2e-steps 1 --steps 10 2>&1 | grep "tcgen05 profile" | tail -2
done
