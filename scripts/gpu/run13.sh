python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
mkdir -p gpurun_out/r13
timeout 300 python -m pytest -q --timeout 300 tests/test_gpu_tall.py > gpurun_out/r13/pytest_tall.log 2>&1; tail -2 gpurun_out/r13/pytest_tall.log
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r13/bench_c5.json 2> gpurun_out/r13/bench_c5.err
tail -c 300 gpurun_out/r13/bench_c5.json
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r13/launches_decompose_c5.csv python scripts/prof_decompose.py c5 > gpurun_out/r13/prof_decompose_c5.log 2>&1
timeout 900 python -m pytest -q --timeout 600 tests/test_gpu_parity.py -k "c5 or c2 or c3" tests/test_gpu_parity_full.py > gpurun_out/r13/pytest.log 2>&1; tail -3 gpurun_out/r13/pytest.log
