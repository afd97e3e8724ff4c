timeout 120 python scripts/bench_jacobi.py 2>&1 | tail -6
timeout 900 python -m pytest tests/ -m gpu -x -q -k "decompose or small_svd or jacobi or edge or c3_noiseless" > gpurun_out/pytest_q.log 2>&1; echo "pytest $?"; tail -2 gpurun_out/pytest_q.log
timeout 900 python scripts/sweep_warm.py c1,c2,c3,c4 d d
