set -x
timeout 600 python -m pytest tests/test_gpu_tc.py -x -q > gpurun_out/pytest_tc.log 2>&1; echo "pytest tc exit $?"
tail -15 gpurun_out/pytest_tc.log
for c in c2 c3; do timeout 300 python scripts/bench_products.py $c tc,fft 32 20; done > gpurun_out/prod_paths4.log 2>&1
cat gpurun_out/prod_paths4.log
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_tc4.csv python scripts/bench_products.py c2 tc,fft 32 3 > /dev/null 2>&1
python scripts/launch_summary.py gpurun_out/launches_tc4.csv | head -12
python scripts/bench_products.py c2 tc 32 3 > gpurun_out/plain_tc.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:hankel_tc -c 2 -o gpurun_out/prof_tc4_c2 python scripts/bench_products.py c2 tc 32 3 > gpurun_out/ncu_tc_c2.log 2>&1
echo "ncu $?"
