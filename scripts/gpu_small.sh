timeout 300 python scripts/bench_tall.py 2>&1 | grep "upd  M=     [14]0"
SSA_SPLIT_OFF=1 timeout 300 python scripts/bench_tall.py 2>&1 | grep "upd  M=     [14]0"
timeout 500 python -m pytest tests/test_gpu_tall.py -q 2>&1 | tail -2
timeout 900 python -m pytest tests/ -m gpu -x -q -k "decompose or edge or c1" > gpurun_out/pytest_q.log 2>&1; echo "pytest $?"; tail -2 gpurun_out/pytest_q.log
timeout 900 python scripts/sweep_warm.py c1,c2,c3 d d
