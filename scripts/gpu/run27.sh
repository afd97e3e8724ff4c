python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
mkdir -p gpurun_out/r27
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r27/smoke.log 2>&1; tail -1 gpurun_out/r27/smoke.log
timeout 900 python bench.py > gpurun_out/r27/bench_c5.json 2> gpurun_out/r27/bench_c5.err
python - <<'P'
import json; d=json.loads(open('gpurun_out/r27/bench_c5.json').read().strip().splitlines()[-1])
print({k: d.get(k) for k in ('value','ms_per_step','rank_r_time_ms')}, d.get('phases_device_ms'), d['roofline']['frac'], d['decomposition'])
P
for c in c2 c3 c4; do timeout 600 python bench.py --config $c --no-cpu-baseline > gpurun_out/r27/bench_$c.json 2> gpurun_out/r27/bench_$c.err; python -c "import json; d=json.loads(open('gpurun_out/r27/bench_$c.json').read().strip().splitlines()[-1]); print('$c', d['ms_per_step'], d.get('rank_r_time_ms'))"; done
timeout 1800 python -m pytest tests -m gpu -q --timeout 900 -x > gpurun_out/r27/pytest_gpu.log 2>&1
tail -5 gpurun_out/r27/pytest_gpu.log
