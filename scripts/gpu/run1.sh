set -x
nvidia-smi --query-gpu=name,clocks.sm --format=csv
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 tests/test_gpu_parity_full.py > gpurun_out/pytest_full.log 2>&1
timeout 300 python scripts/measure_tau.py fft,tc,direct > gpurun_out/tau.json 2> gpurun_out/tau.err
timeout 900 python -m pytest tests -m gpu -q --timeout 600 --deselect tests/test_gpu_parity_full.py > gpurun_out/pytest_rest.log 2>&1
tail -3 gpurun_out/pytest_full.log gpurun_out/pytest_rest.log
cat gpurun_out/tau.err
