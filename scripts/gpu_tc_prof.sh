set -x
python scripts/bench_products.py c2 tc 32 3 > gpurun_out/plain_tc.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:hankel_tc -c 2 -o gpurun_out/prof_tc_c2 python scripts/bench_products.py c2 tc 32 3 > gpurun_out/ncu_tc_c2.log 2>&1
echo "ncu1 $?"
python scripts/bench_products.py c3 tc 32 3 > gpurun_out/plain_tc3.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:hankel_tc -s 1 -c 1 -o gpurun_out/prof_tc_c3 python scripts/bench_products.py c3 tc 32 3 > gpurun_out/ncu_tc_c3.log 2>&1
echo "ncu2 $?"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_tc_c2.csv python scripts/bench_products.py c2 tc,fft 32 3 > /dev/null 2>&1
echo "ncu3 $?"
