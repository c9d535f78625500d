# int8 engine (ticketed units): DRAM traffic / L2 hit / time vs the band (MHAR_I8_GROUP)
mkdir -p gpurun_out
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct
for g in ${GS:-1 4 8 16}; do
  MHAR_I8_GROUP=$g ncu --metrics $M --clock-control none -k regex:chord_i8 --launch-skip 2 -c 1 \
      --csv --log-file gpurun_out/i8g_$g.csv python bench.py --f64-engine int8 --steps 4 \
      --warmup 3 --no-cpu --no-fp32 --no-i8 --e2e-steps 1 > /dev/null 2>&1
  for i in 1 2; do
  MHAR_I8_GROUP=$g python bench.py --f64-engine int8 --steps 10 --no-cpu --no-fp32 --no-i8 \
      --e2e-steps 1 2>/dev/null | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('group $g', round(d['roofline']['avg_launch_ms'],3), d['clocks']['sm_mhz'], round(d['value']))"
  done
done
