echo NC16; timeout 120 python scripts/bench_jacobi.py 2>&1 | tail -6
echo NC32; SSA_JACOBI_NC=32 timeout 120 python scripts/bench_jacobi.py 2>&1 | tail -6
