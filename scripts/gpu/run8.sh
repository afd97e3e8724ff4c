python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
for c in c3 c4 c5; do timeout 300 python scripts/time_products.py $c 0 10; done > gpurun_out/tp8.log 2>&1
cat gpurun_out/tp8.log
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:rpass --csv --log-file gpurun_out/launch8_c5.csv python scripts/time_products.py c5 0 1 > /dev/null 2>&1
timeout 600 python -m pytest -q --timeout 600 tests/test_gpu_parity.py -k "products or reconstruct or c3" > gpurun_out/pytest8.log 2>&1
tail -3 gpurun_out/pytest8.log
