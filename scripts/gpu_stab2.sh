timeout 900 python -m pytest tests/ -m gpu -x -q -k "fft and not c5" > gpurun_out/pytest_q.log 2>&1; echo "pytest $?"; tail -2 gpurun_out/pytest_q.log
for a in "c2 fft 32" "c3 fft 32" "c5 fft 64"; do python scripts/bench_products.py $a 3 2>&1 | tail -2; done
