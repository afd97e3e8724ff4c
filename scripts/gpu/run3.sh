set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
for c in c3 c4 c5; do
  timeout 300 python scripts/time_products.py $c 0 10 >> gpurun_out/tp_new.log 2>&1
  SSA_FFT_STOCKHAM=1 timeout 300 python scripts/time_products.py $c 0 10 >> gpurun_out/tp_old.log 2>&1
done
cat gpurun_out/tp_new.log gpurun_out/tp_old.log
timeout 900 python -m pytest -q --timeout 600 tests/test_gpu_parity_full.py -k "c5 or uv" tests/test_gpu_parity.py -k "band or wcor or c5 or errors or uv" > gpurun_out/pytest3.log 2>&1
tail -15 gpurun_out/pytest3.log
SSA_FFT_STOCKHAM=1 timeout 600 python -m pytest -q --timeout 600 tests/test_gpu_parity_full.py -k c5 > gpurun_out/pytest3_old.log 2>&1
tail -8 gpurun_out/pytest3_old.log
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
tail -c 3000 gpurun_out/bench_c5.json; tail -5 gpurun_out/bench_c5.err
