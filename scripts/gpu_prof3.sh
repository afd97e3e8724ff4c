python scripts/bench_tall1.py 0 201601 224 32 && ncu --set full --import-source on --clock-control none -k regex:gram_tc3 -s 1 -c 1 -o gpurun_out/prof_gram_tc3_c3 -f python scripts/bench_tall1.py 0 201601 224 32 > gpurun_out/ncu_a.log 2>&1; echo "rc $?"
python scripts/bench_tall1.py 1 201601 224 32 && ncu --set full --import-source on --clock-control none -k regex:update_tc2 -s 1 -c 1 -o gpurun_out/prof_update_tc2_c3 -f python scripts/bench_tall1.py 1 201601 224 32 > gpurun_out/ncu_b.log 2>&1; echo "rc $?"
python scripts/bench_tall1.py 0 1844160 356 64 && ncu --set full --import-source on --clock-control none -k regex:gram_tc3 -s 1 -c 1 -o gpurun_out/prof_gram_tc3_c5 -f python scripts/bench_tall1.py 0 1844160 356 64 > gpurun_out/ncu_c.log 2>&1; echo "rc $?"
for f in prof_gram_tc3_c3 prof_update_tc2_c3 prof_gram_tc3_c5; do ncu -i gpurun_out/$f.ncu-rep --page details --csv > gpurun_out/$f.details.csv 2>/dev/null; done
ls -la gpurun_out/*.ncu-rep
