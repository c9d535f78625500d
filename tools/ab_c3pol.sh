# chord3 L2 policies (A_I stream / direction tiles): DRAM bytes, L2 hit rate
# and launch time at config 5 (ncu metrics pass, then an un-profiled bench)
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct
for v in a0d0 a1d0 a0d1 a1d1; do
  MHAR_LIB=tools/ab_$v.so ncu --metrics $M --clock-control none -k regex:chord3_kernel --launch-skip 2 -c 1 \
      --csv --log-file gpurun_out/pol_$v.csv python bench.py --config 5 --steps 4 --warmup 3 \
      --no-cpu --no-fp32 --no-i8 --e2e-steps 1 > /dev/null 2>&1
  MHAR_LIB=tools/ab_$v.so python bench.py --config 5 --steps 10 --no-cpu --no-fp32 --no-i8 \
      --e2e-steps 1 2>/dev/null | tail -1 > gpurun_out/pol_$v.json
done
