timeout 900 python -m pytest tests/ -m gpu -x -q -k "fft or edge or mssa or c2" > gpurun_out/pytest_q.log 2>&1; echo "pytest $?"; tail -2 gpurun_out/pytest_q.log
python scripts/bench_products.py c2 fft 32 3 2>&1 | tail -2
SSA_FFT_NOFOLD=1 python scripts/bench_products.py c2 fft 32 3 2>&1 | tail -2
timeout 900 python scripts/sweep_warm.py c2 d d
python bench.py --steps 5 --warmup 3 --config c2 --no-cpu-baseline > gpurun_out/bg_c2.json 2>/dev/null; python -c "import json;d=json.load(open('gpurun_out/bg_c2.json'));print(d['ms_per_step'], d['value'], d['roofline']['frac'], d['roofline']['avg_launch_ms'], d['config']['path'])"
