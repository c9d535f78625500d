# DRAM traffic / L2 hit rate / time of the DMMA incremental chord kernel ($K, default chord3_kernel) against the
# rasterisation band height (MHAR_GROUP_M row tiles per band), config $CFG
mkdir -p gpurun_out
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct
for g in ${GS:-4 8 16 32}; do
  MHAR_GROUP_M=$g ncu --metrics $M --clock-control none -k regex:${K:-chord3_kernel} --launch-skip 2 -c 1 \
      --csv --log-file gpurun_out/gm_c${CFG:-5}_$g.csv python bench.py --config ${CFG:-5} --steps 4 \
      --warmup 3 --no-cpu --no-fp32 --no-i8 --e2e-steps 1 > /dev/null 2>&1
  MHAR_GROUP_M=$g python bench.py --config ${CFG:-5} --steps 10 --no-cpu --no-fp32 --no-i8 \
      --e2e-steps 3 2>/dev/null | tail -1 > gpurun_out/gm_c${CFG:-5}_$g.json
done
