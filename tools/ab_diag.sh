# diag_chord_kernel occupancy / grid: whole-iterate time on mid-size bodies
for v in "tools/ab_diag1.so 1" "tools/ab_diag1.so 2" "tools/ab_diag1.so 4" "tools/ab_diag2.so 2" "tools/ab_diag2.so 4" "tools/ab_diag2.so 8"; do
  set -- $v
  for b in "hypercube 5000 1000" "simplex 5000 1000" "hypercube 2500 1500"; do
    echo "$1 ctas=$2 $(MHAR_LIB=$1 MHAR_DIAG_CTAS=$2 python tools/mid_body_probe.py $b 100)"
  done
done
