#!/bin/bash
out=gpurun_out/s22; mkdir -p $out
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1 || { tail -20 $out/build.log; exit 1; }
for c in c5 c5 c3 c4; do timeout 300 python scripts/prof_products.py $c fft 2>&1 | tail -2; done
timeout 900 python -m pytest tests -m gpu -q -x -k "product or recon or fft or sigma" --timeout 600 > $out/pytest.log 2>&1; tail -2 $out/pytest.log
timeout 600 python bench.py --no-cpu-baseline > $out/bench_c5.json 2> $out/bench_c5.err
python -c "import json; d=json.loads(open('$out/bench_c5.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['step_ms'], d.get('rank_r_time_ms'), d['roofline']['frac'], {k: v['avg_launch_ms'] for k, v in d['roofline']['products'].items()})"
