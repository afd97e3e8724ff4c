for e in 1e-4 3e-4 1e-3; do echo "EARLY=$e"; SSA_JACOBI_EARLY=$e timeout 900 python scripts/sweep_warm.py c2,c3,c4 d d; done
SSA_JACOBI_EARLY=1e-3 timeout 900 python -m pytest tests/ -m gpu -x -q -k "decompose or c3_noiseless or edge" 2>&1 | tail -2
