python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
mkdir -p gpurun_out/r11
for c in c3 c4 c5; do timeout 300 python scripts/time_products.py $c 0 10; done > gpurun_out/r11/tp.log 2>&1
cat gpurun_out/r11/tp.log
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:rpass --csv --log-file gpurun_out/r11/launch_c5.csv python scripts/time_products.py c5 0 1 > /dev/null 2>&1
timeout 600 python -m pytest -q --timeout 600 tests/test_gpu_parity.py -k "products or c3 or c2" > gpurun_out/r11/pytest.log 2>&1
tail -3 gpurun_out/r11/pytest.log
