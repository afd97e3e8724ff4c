#!/bin/bash
# Round validation on one B200 (run through gpurun from the repo root):
#   build, smoke, bench c5 (default) + c1..c4, the GPU test suite, the c5 ncu launch list, the ncu DRAM
#   traffic of one block product per config (roofline.traffic) and an ncu --set full of c5's products.
# Usage: bash scripts/gpu_validate.sh <tag> [quick]
tag=${1:-val}; out=gpurun_out/$tag; mkdir -p $out
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1 || { tail -20 $out/build.log; exit 1; }
python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1; tail -1 $out/smoke.log
# traffic first: bench reads profiles/<round>/traffic.json, refreshed from these captures
for c in c2 c3 c4 c5; do for w in xv xtu; do
  timeout 600 ncu --profile-from-start off --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
    --csv --log-file $out/traffic_${c}_$w.csv python scripts/traffic_products.py $c $w > /dev/null 2>&1
done; done
python scripts/traffic_summary.py $out/traffic_c*_*.csv > $out/traffic.json && cp $out/traffic.json profiles/r02/traffic.json
timeout 900 python bench.py > $out/bench_c5.json 2> $out/bench_c5.err
python - "$out" <<'P'
import json, sys
d = json.loads(open(sys.argv[1] + '/bench_c5.json').read().strip().splitlines()[-1])
print({k: d.get(k) for k in ('value', 'ms_per_step', 'rank_r_time_ms', 'step_ms')}, d.get('phases_device_ms'),
      d['roofline']['frac'], d['roofline'].get('traffic'), d['roofline'].get('step_shares'))
P
for c in c1 c2 c3 c4; do
  timeout 600 python bench.py --config $c --no-cpu-baseline > $out/bench_$c.json 2> $out/bench_$c.err
  python -c "import json; d=json.loads(open('$out/bench_$c.json').read().strip().splitlines()[-1]); print('$c', d['ms_per_step'], d.get('rank_r_time_ms'), d['roofline']['frac'])"
done
timeout 900 python bench.py --impl reference --steps 2 --warmup 3 > $out/bench_ref.json 2> $out/bench_ref.err
# the N = 2 command on one GPU (gloo, all ranks on cuda:0): correctness rehearsal, not a measurement
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29517 \
  bench.py --gpus 2 --one-gpu-rehearsal --steps 2 --warmup 3 > $out/bench_c5_rehearsal_n2.json 2> $out/bench_c5_rehearsal_n2.err
python -c "import json; d=json.loads([l for l in open('$out/bench_c5_rehearsal_n2.json') if l.startswith('{')][-1]); print('rehearsal n2', d['ms_per_step'], d['sigma_head'], d['decomposition'])"
[ "$2" = quick ] && exit 0
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 > $out/pytest_gpu.log 2>&1
tail -3 $out/pytest_gpu.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file $out/launches_bench_c5.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $out/ncu_bench.log 2>&1
python scripts/launch_summary.py $out/launches_bench_c5.csv > $out/launches_bench_c5.summary.txt 2>&1; head -12 $out/launches_bench_c5.summary.txt
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:rpass_ --launch-skip 6 --launch-count 6 \
  -o $out/prof_rpass_c5 python scripts/prof_products.py c5 fft 64 1 > $out/ncu_rpass.log 2>&1
python scripts/ncu_brief.py $out/prof_rpass_c5.ncu-rep > $out/prof_rpass_c5.summary.txt 2>&1; cat $out/prof_rpass_c5.summary.txt
