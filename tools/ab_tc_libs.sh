# fp32 variant: ncu DRAM traffic + bench launch time per engine build (LIBS), both direction forms
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct
for lib in ${LIBS:-tools/ab_base.so}; do
  for dir in split rounded; do
    MHAR_LIB=$lib ncu --metrics $M --clock-control none -k regex:chord_tc32 --launch-skip 2 -c 1 --csv \
      --log-file gpurun_out/tc_$(basename $lib .so)_$dir.csv python bench.py --precision 32 --fp32-direction $dir \
      --steps 4 --warmup 3 --no-cpu --no-fp32 --no-i8 --e2e-steps 1 > /dev/null 2>&1
  done
done
for i in 1 2; do
  for lib in ${LIBS:-tools/ab_base.so}; do
    for dir in split rounded; do
      MHAR_LIB=$lib timeout 300 python bench.py --precision 32 --fp32-direction $dir --no-i8 --no-fp32 --no-cpu --e2e-steps 1 --steps 10 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read().splitlines()[-1]);print('$lib $dir', round(d['roofline']['avg_launch_ms'],3), d['clocks']['sm_mhz'], round(d['value']))"
    done
  done
done
