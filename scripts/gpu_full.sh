set -x
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?"
tail -4 gpurun_out/pytest_gpu.log
python bench.py --steps 5 --warmup 3 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo "bench c2 exit $?"
for c in c1 c3 c4; do python bench.py --steps 3 --warmup 3 --config $c --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo "bench $c exit $?"; done
SSA_ORTH_FAST=1 python bench.py --steps 3 --warmup 3 --config c2 --no-cpu-baseline > gpurun_out/bench_c2_fast.json 2>&1; echo "fast $?"
SSA_ORTH_FAST=1 python bench.py --steps 3 --warmup 3 --config c3 --no-cpu-baseline > gpurun_out/bench_c3_fast.json 2>&1; echo "fast3 $?"
