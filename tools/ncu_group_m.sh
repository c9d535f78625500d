# DRAM traffic of the DMMA chord kernel vs the rasterisation band height
mkdir -p gpurun_out
for g in ${GS:-1 2 4 8 32}; do
  MHAR_GROUP_M=$g ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:chord2_kernel --launch-skip 1 -c 1 --csv --log-file gpurun_out/gm_$g.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-fp32 --no-i8 --e2e-steps 1 > /dev/null 2>&1
done
