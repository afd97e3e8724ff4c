for t in 1e-12 1e-10 1e-9 1e-8; do echo "tol $t"; SSA_JACOBI_TOL=$t python scripts/sweep_k.py c3 32 4; SSA_JACOBI_TOL=$t python scripts/sweep_k.py c2 16 4; done
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -k "decompose or noiseless or wcor" > gpurun_out/pytest_tol.log 2>&1; echo "pytest $?"; tail -2 gpurun_out/pytest_tol.log
