set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 900 python -m pytest -q --timeout 600 tests/test_gpu_parity_full.py -k "c5" > gpurun_out/pytest4.log 2>&1
tail -4 gpurun_out/pytest4.log
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:rpass --csv --log-file gpurun_out/launch_c5.csv python scripts/time_products.py c5 0 1 > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:rpass --csv --log-file gpurun_out/launch_c3.csv python scripts/time_products.py c3 0 1 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:rpass --launch-skip 6 -c 6 -o gpurun_out/prof_rfft_c5 python scripts/time_products.py c5 0 1 > gpurun_out/ncu_full.log 2>&1
tail -3 gpurun_out/ncu_full.log
