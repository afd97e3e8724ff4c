set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
for c in c2 c3 c4 c5; do timeout 300 python scripts/time_products.py $c 0 10; done > gpurun_out/tp6.log 2>&1
cat gpurun_out/tp6.log
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:rpass --csv --log-file gpurun_out/launch6_c5.csv python scripts/time_products.py c5 0 1 > /dev/null 2>&1
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/bench6_c5.json 2> gpurun_out/bench6_c5.err
tail -c 1500 gpurun_out/bench6_c5.json
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/pytest6.log 2>&1
tail -12 gpurun_out/pytest6.log
