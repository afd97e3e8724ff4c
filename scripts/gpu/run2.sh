set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "products" > gpurun_out/pytest_products.log 2>&1
tail -5 gpurun_out/pytest_products.log
for c in c3 c4 c5; do
  timeout 300 python scripts/bench_products.py $c fft 0 10 >> gpurun_out/prod_new.log 2>&1
  SSA_FFT_STOCKHAM=1 timeout 300 python scripts/bench_products.py $c fft 0 10 >> gpurun_out/prod_old.log 2>&1
done
cat gpurun_out/prod_new.log gpurun_out/prod_old.log
timeout 1200 python -m pytest tests/test_gpu_parity_full.py -q --timeout 900 > gpurun_out/pytest_full.log 2>&1
tail -15 gpurun_out/pytest_full.log
timeout 1200 python -m pytest tests -m gpu -q --timeout 900 --ignore tests/test_gpu_parity_full.py > gpurun_out/pytest_rest.log 2>&1
tail -15 gpurun_out/pytest_rest.log
