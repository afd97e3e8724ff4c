for k in 32 16 64; do echo "k$k"; timeout 60 python scripts/tc_debug.py $k 2>&1 | tail -1; done
timeout 600 python -m pytest tests/test_gpu_tc.py -x -q > gpurun_out/pytest_tc.log 2>&1; echo "pytest tc exit $?"
tail -3 gpurun_out/pytest_tc.log
timeout 300 python scripts/bench_products.py c2 tc,fft 32 20 > gpurun_out/prod_paths8.log 2>&1; cat gpurun_out/prod_paths8.log
python scripts/bench_products.py c2 tc 32 3 > gpurun_out/plain_tc.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_tc8.csv python scripts/bench_products.py c2 tc 32 3 > /dev/null 2>&1 && python scripts/launch_summary.py gpurun_out/launches_tc8.csv | head -6
python scripts/bench_products.py c2 tc 32 3 > gpurun_out/plain_tc.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:hankel_tc -c 2 -o gpurun_out/prof_tc8_c2 python scripts/bench_products.py c2 tc 32 3 > gpurun_out/ncu_tc_c2.log 2>&1
echo "ncu $?"
