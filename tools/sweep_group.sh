#!/bin/bash
# Chord-kernel rasterisation sweep: device time and DRAM bytes per launch.
for g in 2 4 8 16; do
  MHAR_GROUP_M=$g python bench.py --steps 6 --warmup 3 --no-cpu --e2e-steps 1 > gpurun_out/sweep_g$g.json 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/sweep_g$g.json').read().strip().splitlines()[-1]);print('group_m',$g,'value',round(d['value']),'frac',round(d['roofline']['frac'],4),'chord_ms',round(d['roofline']['avg_launch_ms'],2))"
done
