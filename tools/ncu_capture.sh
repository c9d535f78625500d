# ncu captures behind profiles/ncu_full_rNN.json and profiles/ncu_launches_rNN.csv:
# one --set full capture per tensor-core kernel (config 5, 4096 walks, an
# incremental launch after the warm-up), then the launch list of a short bench run.
set -x
mkdir -p gpurun_out
B="--steps 4 --warmup 3 --no-cpu --no-fp32 --no-i8 --e2e-steps 1"
ncu --set full --clock-control none --import-source on -k regex:chord3_kernel --launch-skip 2 -c 1 -f -o gpurun_out/chord3_full python bench.py $B > gpurun_out/ncu_full64.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:chord3_kernel --launch-skip 2 -c 1 -f -o gpurun_out/chord3_c3_full python bench.py --config 3 $B > gpurun_out/ncu_full64c3.log 2>&1
MHAR_CHORD3=0 ncu --set full --clock-control none --import-source on -k regex:chord2_kernel --launch-skip 2 -c 1 -f -o gpurun_out/chord2_full python bench.py $B > gpurun_out/ncu_full64c2.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:chord_tc32 --launch-skip 2 -c 1 -f -o gpurun_out/tc32_full python bench.py --precision 32 $B > gpurun_out/ncu_full32.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:chord_tc32 --launch-skip 2 -c 1 -f -o gpurun_out/tc32r_full python bench.py --precision 32 --fp32-direction rounded $B > gpurun_out/ncu_full32r.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:chord_i8 --launch-skip 2 -c 1 -f -o gpurun_out/i8_full python bench.py --f64-engine int8 $B > gpurun_out/ncu_i8.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu --e2e-steps 1 > gpurun_out/ncu_launch.log 2>&1
ls -la gpurun_out/*.ncu-rep
