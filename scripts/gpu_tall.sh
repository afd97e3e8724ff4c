echo NEW; timeout 300 python scripts/bench_tall.py 2>&1 | tail -8
echo OLD; SSA_UPD_OLD=1 timeout 300 python scripts/bench_tall.py 2>&1 | tail -8
timeout 900 python -m pytest tests/ -m gpu -x -q -k "decompose or edge or reconstruct or band or c3_noiseless" > gpurun_out/pytest_q.log 2>&1; echo "pytest $?"; tail -3 gpurun_out/pytest_q.log
for c in c2 c3; do python bench.py --steps 5 --warmup 3 --config $c --no-cpu-baseline > gpurun_out/bg_$c.json 2> gpurun_out/bg_$c.err; echo "bench $c $?"; python -c "import json;d=json.load(open('gpurun_out/bg_$c.json'));print(d['ms_per_step'], d['decomposition']['ms_ritz_per_step'], d['decomposition']['n_restarts'], d['decomposition']['n_block_products'])"; done
