# DRAM traffic, L2 hit rate and time of the DMMA incremental chord kernel
# (chord2_kernel<INCREMENTAL>) at BASELINE configs 5 and 3: one launch each
# after the refresh, metrics only (replayed by ncu; the times are not bench numbers).
mkdir -p gpurun_out
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active
for cfg in ${CFGS:-5 3}; do
  ncu --metrics $M --clock-control none -k regex:chord2_kernel --launch-skip 2 -c 1 --csv \
      --log-file gpurun_out/traffic_c$cfg.csv python bench.py --config $cfg --steps 4 --warmup 3 \
      --no-cpu --no-fp32 --no-i8 --e2e-steps 1 > /dev/null 2>&1
done
