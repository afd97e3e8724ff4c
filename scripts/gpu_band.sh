timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "band" > gpurun_out/pytest_band.log 2>&1; echo "pytest $?"; tail -15 gpurun_out/pytest_band.log
