# Round-2 re-measure on one box: smoke, GPU tests, bench lines (configs 5/3/4, reference arm), ncu captures
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f_smoke.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/f_tests.log 2>&1; echo rc=$? >> gpurun_out/f_tests.log
python bench.py > gpurun_out/f_bench5.log 2>&1
python bench.py --config 3 --no-cpu > gpurun_out/f_bench3.log 2>&1
python bench.py --config 4 --no-cpu > gpurun_out/f_bench4.log 2>&1
python bench.py --impl reference > gpurun_out/f_ref.log 2>&1
bash tools/ncu_capture.sh > gpurun_out/f_ncu.log 2>&1
# summarise the captures on the box (gpurun_out/ travels back only under 64 MiB)
MHAR_CAPTURE_COMMIT=${MHAR_CAPTURE_COMMIT:-unknown} python tools/ncu_summarize.py gpurun_out/ncu_full_r02.json > gpurun_out/f_ncu_summary.log 2>&1
cp gpurun_out/launches.csv gpurun_out/ncu_launches_r02.csv 2>/dev/null
rm -f gpurun_out/chord2_full.ncu-rep gpurun_out/tc32_full.ncu-rep gpurun_out/tc32r_full.ncu-rep gpurun_out/i8_full.ncu-rep gpurun_out/chord3_full.ncu-rep
