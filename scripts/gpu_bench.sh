#!/bin/bash
# Bench c5 (+ optional configs) and the FFT product parity tests on one B200.
# Usage: bash scripts/gpu_bench.sh <tag> [configs...]
tag=${1:-bench}; shift; out=gpurun_out/$tag; mkdir -p $out
for c in c5 "$@"; do
  timeout 900 python bench.py --config $c $([ $c != c5 ] && echo --no-cpu-baseline) > $out/bench_$c.json 2> $out/bench_$c.err
  python - $out/bench_$c.json <<'P'
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
r = d['roofline']
print(d['config']['workload'], 'ms/step', round(d['ms_per_step'], 2), 'rank_r', round(d.get('rank_r_time_ms', 0), 2), d.get('phases_device_ms', {}).get('reconstruct'),
      'frac', round(r['frac'], 3), {k: round(v['avg_launch_ms'], 3) for k, v in r.get('products', {}).items()}, r.get('step_shares'))
P
done
