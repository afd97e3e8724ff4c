set -x
timeout 120 python scripts/bench_products.py c2 tc 32 5 > gpurun_out/tc_c2_first.log 2>&1; echo "first exit $?"
cat gpurun_out/tc_c2_first.log | tail -5
timeout 600 python -m pytest tests/test_gpu_tc.py -x -q > gpurun_out/pytest_tc.log 2>&1; echo "pytest tc exit $?"
tail -30 gpurun_out/pytest_tc.log
for c in c2 c3 c4; do timeout 300 python scripts/bench_products.py $c tc,fft,direct 32 20; done > gpurun_out/prod_paths.log 2>&1
cat gpurun_out/prod_paths.log
