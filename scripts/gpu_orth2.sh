for c in c2 c3 c1 c4; do SSA_DEBUG=1 python scripts/debug_decompose.py $c auto 2>&1 | grep -E "host ms|^c[0-9]" | tail -2; done
for c in c2 c3; do SSA_ORTH_LEGACY=1 SSA_DEBUG=1 python scripts/debug_decompose.py $c auto 2>&1 | grep -E "host ms" | tail -1; done
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_tc.py -x -q > gpurun_out/pytest_o2.log 2>&1; echo "pytest $?"; tail -3 gpurun_out/pytest_o2.log
