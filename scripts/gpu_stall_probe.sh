#!/bin/bash
# Probe of one-off host/GPU stalls in the first bench process after other GPU activity (gpurun r2/r3):
# the multi-rank rehearsal test recreates the "busy box" state, then bench c5 runs with the clock sampler,
# without it (SSA_BENCH_NO_CLOCKS=1) and with the solver's phase timings (SSA_DEBUG=1).
out=gpurun_out/${1:-probe}; mkdir -p $out
show() { python -c "import json,sys; d=json.loads(open('$1').read().strip().splitlines()[-1]); print('$1', d['step_ms'], d['e2e']['step_ms'], d['clocks'])"; }
busy() { timeout 900 python -m pytest tests/test_gpu_bench_ranks.py -x -q --timeout 800 -k "c5" > $out/busy_$1.log 2>&1; tail -1 $out/busy_$1.log; }
busy 1
timeout 600 python bench.py --no-cpu-baseline > $out/A1.json 2> $out/A1.err; show $out/A1.json
timeout 600 python bench.py --no-cpu-baseline > $out/A2.json 2> $out/A2.err; show $out/A2.json
busy 2
SSA_BENCH_NO_CLOCKS=1 timeout 600 python bench.py --no-cpu-baseline > $out/B1.json 2> $out/B1.err; show $out/B1.json
busy 3
SSA_DEBUG=1 timeout 600 python bench.py --no-cpu-baseline > $out/D1.json 2> $out/D1.err; show $out/D1.json
busy 4
timeout 600 python bench.py --no-cpu-baseline > $out/A3.json 2> $out/A3.err; show $out/A3.json
