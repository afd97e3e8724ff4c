#!/bin/bash
out=gpurun_out/s18; mkdir -p $out
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1 || { tail -20 $out/build.log; exit 1; }
timeout 600 python -m pytest tests/test_gpu_tall.py -q -x > $out/pytest_tall.log 2>&1; tail -2 $out/pytest_tall.log
for sp in 1 0 1; do
SSA_GRAM_SPLIT=$sp timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > $out/bench_c5_$sp.json 2> $out/bench_c5_$sp.err
python -c "import json; d=json.loads(open('$out/bench_c5_$sp.json').read().strip().splitlines()[-1]); print('split=$sp', round(d['ms_per_step'],2), round(d.get('rank_r_time_ms'),2), d['step_ms'], d['decomposition']['max_rel_residual'])" 2>&1 | tail -1
done
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 900 > $out/pytest_gpu.log 2>&1
tail -3 $out/pytest_gpu.log
