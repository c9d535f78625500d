for cfg in 3 5; do
  MHAR_C3_PROFILE=1 timeout 300 python bench.py --config $cfg --no-i8 --no-fp32 --no-cpu --e2e-steps 1 --steps 10 > gpurun_out/prof_c$cfg.json 2> gpurun_out/prof_c$cfg.err
done
