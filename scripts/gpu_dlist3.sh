for c in c2 c3 c4 c5; do
python scripts/prof_decompose.py $c > gpurun_out/pd_$c.log 2>&1 && ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_dec_$c.csv python scripts/prof_decompose.py $c > /dev/null 2>&1; echo "$c $?"; cat gpurun_out/pd_$c.log; python scripts/launch_summary.py gpurun_out/launches_dec_$c.csv | head -14
done
