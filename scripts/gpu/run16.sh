python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
mkdir -p gpurun_out/r16
for c in c3 c5; do timeout 300 python scripts/time_products.py $c 0 10; done
timeout 900 ncu --set full --import-source on --clock-control none -k regex:rpass -c 6 -o gpurun_out/r16/rfft_c5 python scripts/time_products.py c5 0 1 > gpurun_out/r16/ncu_c5.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:rpass -c 6 -o gpurun_out/r16/rfft_c3 python scripts/time_products.py c3 0 1 > gpurun_out/r16/ncu_c3.log 2>&1
tail -3 gpurun_out/r16/ncu_c5.log
