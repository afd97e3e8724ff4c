timeout 900 python -m pytest tests/test_gpu_edge.py -q > gpurun_out/pytest_edge.log 2>&1; echo "pytest $?"; grep -E "passed|failed|Error|assert" gpurun_out/pytest_edge.log | head -30
