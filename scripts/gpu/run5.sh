set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
for c in c3 c4 c5; do timeout 300 python scripts/time_products.py $c 0 10; done > gpurun_out/tp5.log 2>&1
cat gpurun_out/tp5.log
timeout 900 python -m pytest -q --timeout 600 tests/test_gpu_parity.py -k "products or band or c5 or decompose_c2" tests/test_gpu_parity_full.py -k "c5 or c3" > gpurun_out/pytest5.log 2>&1
tail -5 gpurun_out/pytest5.log
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:rpass --csv --log-file gpurun_out/launch5_c5.csv python scripts/time_products.py c5 0 1 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:rpass --launch-skip 6 -c 6 -o gpurun_out/prof5_c5 python scripts/time_products.py c5 0 1 > gpurun_out/ncu5.log 2>&1
tail -2 gpurun_out/ncu5.log
