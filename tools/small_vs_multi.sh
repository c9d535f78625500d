# walk-resident small_kernel against the multi-kernel chain on the paper's
# structured bodies: chain-steps/s per (body, n, z); behind the selection rule
# in csrc/abi.cu (MHAR_SMALL_RULE)
for b in ${BODIES:-hypercube simplex}; do for nz in ${NZ:-"1000 1000" "1500 1000" "2000 1000" "2500 1000" "1000 4000" "2500 4000"}; do for m in multi small; do echo "$b $nz $m $(python tools/mid_body_probe.py $b $nz 60 $m | grep -o 'chain_steps_per_s": [0-9.e+]*\|chord_kernel": "[a-z_]*' | tr '\n' ' ')"; done; done; done
