set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "decompose or c3_noiseless or wcor or errors" > gpurun_out/pytest_orth.log 2>&1; echo "pytest exit $?"
tail -5 gpurun_out/pytest_orth.log
for c in c2 c3 c1; do timeout 300 python bench.py --steps 3 --warmup 3 --config $c --no-cpu-baseline > gpurun_out/bo_$c.json 2> gpurun_out/bo_$c.err; echo "bench $c $?"; done
SSA_ORTH_LEGACY=1 timeout 300 python bench.py --steps 3 --warmup 3 --config c2 --no-cpu-baseline > gpurun_out/bo_c2_legacy.json 2>&1
