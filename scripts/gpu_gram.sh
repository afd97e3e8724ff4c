timeout 120 python scripts/bench_jacobi.py 2>&1 | tail -6
timeout 900 python -m pytest tests/ -m gpu -x -q -k "decompose or small_svd or jacobi or c3_noiseless or edge" > gpurun_out/pytest_gram.log 2>&1; echo "pytest $?"; tail -3 gpurun_out/pytest_gram.log
for c in c2 c3; do SSA_DEBUG=1 python scripts/debug_decompose.py $c auto > gpurun_out/dbg_$c.log 2>&1; echo "$c $?"; grep -E "ritz_svd|host ms" gpurun_out/dbg_$c.log | tail -7; done
for c in c2 c3 c4; do python bench.py --steps 5 --warmup 3 --config $c --no-cpu-baseline > gpurun_out/bg_$c.json 2> gpurun_out/bg_$c.err; echo "bench $c $?"; python -c "import json;d=json.load(open('gpurun_out/bg_$c.json'));print(d['ms_per_step'], d['decomposition']['ms_ritz_per_step'], d['decomposition']['n_restarts'])"; done
