for n in 37 74 148 296; do
SSA_TC_CTAS=$n ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/l_$n.csv python scripts/bench_products.py c2 tc 32 3 > /dev/null 2>&1
echo "CTAS $n"; python scripts/launch_summary.py gpurun_out/l_$n.csv | head -4
done
