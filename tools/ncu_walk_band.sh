# DRAM traffic and time of the DMMA chord kernel vs the walk-band rasterisation
mkdir -p gpurun_out
for g in ${GS:-0 8 16 32}; do
  MHAR_WALK_BAND=$g ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:chord2_kernel --launch-skip 1 -c 1 --csv --log-file gpurun_out/wb_$g.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-fp32 --no-i8 --e2e-steps 1 > /dev/null 2>&1
done
for g in ${GS:-0 8 16 32}; do
  MHAR_WALK_BAND=$g timeout 200 python bench.py --no-i8 --no-fp32 --no-cpu --e2e-steps 1 --steps 10 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read().splitlines()[-1]);print('walk_band=$g', round(d['roofline']['avg_launch_ms'],3), round(d['roofline']['frac'],4))"
done
