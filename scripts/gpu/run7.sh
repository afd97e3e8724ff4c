set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
for c in c2 c3 c4 c5; do timeout 300 python scripts/time_products.py $c 0 10; done > gpurun_out/tp7.log 2>&1
cat gpurun_out/tp7.log
timeout 600 python -m pytest -q --timeout 600 tests/test_gpu_param.py > gpurun_out/pytest7p.log 2>&1
tail -15 gpurun_out/pytest7p.log
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:rpass --csv --log-file gpurun_out/launch7_c5.csv python scripts/time_products.py c5 0 1 > /dev/null 2>&1
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -x --ignore tests/test_gpu_param.py > gpurun_out/pytest7.log 2>&1
tail -12 gpurun_out/pytest7.log
