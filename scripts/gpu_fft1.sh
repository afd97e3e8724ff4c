timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "fft" > gpurun_out/pytest_fft.log 2>&1; echo "pytest $?"; tail -3 gpurun_out/pytest_fft.log
for c in c3 c4 c2; do timeout 300 python scripts/bench_products.py $c fft 32 20; done
python scripts/bench_products.py c3 fft 32 3 > gpurun_out/plain_fft.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_fft3.csv python scripts/bench_products.py c3 fft 32 3 > /dev/null 2>&1 && python scripts/launch_summary.py gpurun_out/launches_fft3.csv | head -6
