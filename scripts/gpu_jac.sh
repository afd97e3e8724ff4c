set -x
timeout 120 python scripts/bench_jacobi.py 2>&1 | tail -8
SSA_JACOBI_CLUSTER=1 timeout 120 python scripts/bench_jacobi.py 2>&1 | tail -8
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_tc.py -x -q -k "decompose or c3_noiseless or small_svd or jacobi" > gpurun_out/pytest_jac.log 2>&1; echo "pytest exit $?"
tail -3 gpurun_out/pytest_jac.log
for c in c2 c3 c1 c4; do python bench.py --steps 3 --warmup 3 --config $c --no-cpu-baseline > gpurun_out/bj_$c.json 2> gpurun_out/bj_$c.err; echo "bench $c exit $?"; done
for m in 2 4; do SSA_MCYC=$m python bench.py --steps 3 --warmup 3 --config c2 --no-cpu-baseline > gpurun_out/bj_c2_m$m.json 2>&1; done
SSA_MCYC=3 python bench.py --steps 3 --warmup 3 --config c3 --no-cpu-baseline > gpurun_out/bj_c3_m3.json 2>&1
