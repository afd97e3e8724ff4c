python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
mkdir -p gpurun_out/r10
timeout 600 python -m pytest -q --timeout 600 tests/test_gpu_param.py > gpurun_out/r10/pytest_param.log 2>&1
tail -3 gpurun_out/r10/pytest_param.log
SSA_DEBUG=1 timeout 300 python scripts/debug_decompose.py c5 fft 64 > gpurun_out/r10/debug_c5.log 2>&1
for c in c2 c3 c4 c5; do for pr in xv xtu; do
  ncu --profile-from-start off --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --csv --log-file gpurun_out/r10/traffic_${c}_${pr}.csv python scripts/traffic_products.py $c $pr > /dev/null 2>&1
done; done
for c in c2 c3 c5; do
  ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r10/launches_decompose_$c.csv python scripts/prof_decompose.py $c > gpurun_out/r10/prof_decompose_$c.log 2>&1
done
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r10/bench_c5.json 2> gpurun_out/r10/bench_c5.err
tail -c 300 gpurun_out/r10/bench_c5.json
