timeout 120 python scripts/bench_jacobi.py 2>&1 | tail -6
SSA_JACOBI_BW16=1 timeout 120 python scripts/bench_jacobi.py 2>&1 | tail -6
