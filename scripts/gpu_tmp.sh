#!/bin/bash
out=gpurun_out/s21; mkdir -p $out
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1 || { tail -20 $out/build.log; exit 1; }
for i in 1 2; do
SSA_DEBUG=1 timeout 600 python bench.py --no-cpu-baseline > $out/bench_c5_$i.json 2> $out/bench_c5_$i.err
python -c "import json; d=json.loads(open('$out/bench_c5_$i.json').read().strip().splitlines()[-1]); print('run $i', round(d['ms_per_step'],2), d['step_ms'], d['e2e']['step_ms'], [p[1] for p in d['step_phases_ms']])" 2>&1 | tail -1
grep -E "host ms: products" $out/bench_c5_$i.err | awk '{print $5}' | tr '\n' ';'; echo
done
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 900 > $out/pytest_gpu.log 2>&1
tail -3 $out/pytest_gpu.log
