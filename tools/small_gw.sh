# walk-resident kernel: chain-steps/s against the lanes per walk (MHAR_SMALL_GW)
# on the paper's small hypercubes / simplices; behind small_group_width()
for b in ${BODIES:-"hypercube 3 10000" "hypercube 10 10000" "hypercube 25 5000" "hypercube 50 2500" "simplex 5 10000" "simplex 15 10000" "simplex 25 10000" "simplex 50 10000" "hypercube 100 4000"}; do
  for g in 4 8 16 32; do
    echo "$b gw=$g $(MHAR_SMALL_GW=$g python tools/mid_body_probe.py $b 200 small | grep -o 'chain_steps_per_s": [0-9.e+]*' | tr '\n' ' ')"
  done
done
