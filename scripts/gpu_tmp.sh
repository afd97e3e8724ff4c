#!/bin/bash
out=gpurun_out/s17; mkdir -p $out
for i in 1 2 3; do
SSA_DEBUG=1 timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > $out/bench_c5_$i.json 2> $out/bench_c5_$i.err
python -c "import json; d=json.loads(open('$out/bench_c5_$i.json').read().strip().splitlines()[-1]); print('run $i', round(d['ms_per_step'],2), round(d.get('rank_r_time_ms'),2), d['step_ms'], d['decomposition']['ms_products_per_step'])" 2>&1 | tail -1
grep -E "host ms: products" $out/bench_c5_$i.err | tr '\n' ' ' | cut -c1-400; echo
nvidia-smi --query-gpu=clocks.sm,clocks.mem,power.draw,temperature.gpu --format=csv,noheader
done
