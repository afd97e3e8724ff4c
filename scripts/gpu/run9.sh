python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
mkdir -p gpurun_out/r9
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/r9/bench_c5.json 2> gpurun_out/r9/bench_c5.err
for c in c1 c2 c3 c4; do timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r9/bench_$c.json 2> gpurun_out/r9/bench_$c.err; done
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r9/bench_ref.json 2> gpurun_out/r9/bench_ref.err
for c in c2 c3 c4 c5; do
  ncu --profile-from-start off --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --csv --log-file gpurun_out/r9/traffic_$c.csv python scripts/traffic_products.py $c > /dev/null 2>&1
done
for c in c2 c3 c5; do
  ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r9/launches_decompose_$c.csv python scripts/prof_decompose.py $c > gpurun_out/r9/prof_decompose_$c.log 2>&1
done
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r9/launches_bench_c5.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/r9/ncu_bench.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:rpass --launch-skip 4 -c 8 -o gpurun_out/r9/prof_rfft_c5 python scripts/time_products.py c5 0 1 > gpurun_out/r9/ncu_full.log 2>&1
tail -c 600 gpurun_out/r9/bench_c5.json
