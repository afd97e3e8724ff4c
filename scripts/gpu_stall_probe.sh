#!/bin/bash
# Probe of one-off host stalls in bench c5 steps (gpurun r2: +16..+50 ms in about one step of ten, in 4 of 5
# bench processes, with and without the clock sampler; r3: after bench.py stopped cyclic-GC passes in its
# timed regions).  The multi-rank rehearsal test first recreates a "busy box"; then N bench processes.
out=gpurun_out/${1:-probe}; n=${2:-6}; mkdir -p $out
show() { python -c "import json,sys; d=json.loads(open('$1').read().strip().splitlines()[-1]); print('$1', d['step_ms'], d['e2e']['step_ms'], d.get('step_reconstruct_host_ms'))"; }
timeout 900 python -m pytest tests/test_gpu_bench_ranks.py -x -q --timeout 800 -k "c5" > $out/busy.log 2>&1; tail -1 $out/busy.log
for i in $(seq 1 $n); do
  timeout 600 python bench.py --no-cpu-baseline > $out/A$i.json 2> $out/A$i.err; show $out/A$i.json
done
