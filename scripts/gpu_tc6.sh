SSA_TC_CTAS=37 python scripts/bench_products.py c2 tc 32 3 > gpurun_out/plain_tc.log 2>&1 && \
SSA_TC_CTAS=37 ncu --set full --clock-control none --import-source on -k regex:hankel_tc -c 1 -o gpurun_out/prof_tc37 python scripts/bench_products.py c2 tc 32 3 > gpurun_out/ncu_tc37.log 2>&1
echo "ncu $?"
