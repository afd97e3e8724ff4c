#!/bin/bash
# A/B of one tall-kernel switch: live kernel timings at c5's K side, the tall GPU tests under the
# variant, and the c5 / c3 / c2 bench lines for both settings.
# Usage: bash scripts/gpu_ab_tall.sh <tag> <ENV_NAME> <value_a> <value_b>
tag=${1:-ab}; var=$2; va=$3; vb=$4; out=gpurun_out/$tag; mkdir -p $out
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1 || { tail -20 $out/build.log; exit 1; }
for v in $va $vb; do
  env $var=$v timeout 300 python scripts/bench_tall_c5.py > $out/tall_$v.txt 2>&1
  echo "== $var=$v"; cat $out/tall_$v.txt
done
env $var=$vb timeout 900 python -m pytest tests/test_gpu_tall.py -m gpu -q -x > $out/pytest_tall.log 2>&1; tail -2 $out/pytest_tall.log
for v in $vb $va; do for c in c5 c3 c2; do
  env $var=$v timeout 600 python bench.py --config $c --no-cpu-baseline > $out/bench_${c}_$v.json 2> $out/bench_${c}_$v.err
  python - $out/bench_${c}_$v.json $c $v <<'P'
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(sys.argv[2], '=', sys.argv[3], d['ms_per_step'], d.get('rank_r_time_ms'), d['decomposition']['n_block_products'],
      d['decomposition']['max_rel_residual'], d['roofline']['frac'])
P
done; done
