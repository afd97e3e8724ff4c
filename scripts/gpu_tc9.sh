for k in 32 16 64; do echo "k$k"; timeout 60 python scripts/tc_debug.py $k 2>&1 | tail -1; done
timeout 600 python -m pytest tests/test_gpu_tc.py -x -q > gpurun_out/pytest_tc.log 2>&1; echo "pytest tc exit $?"; tail -2 gpurun_out/pytest_tc.log
python scripts/bench_products.py c2 tc 32 3 > gpurun_out/plain_tc.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_tc9.csv python scripts/bench_products.py c2 tc 32 3 > /dev/null 2>&1 && python scripts/launch_summary.py gpurun_out/launches_tc9.csv | head -6
