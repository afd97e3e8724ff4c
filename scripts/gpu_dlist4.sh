# c2/c3: under ncu every kernel is serialised and slower, which makes the solver's cost-aware
# convergence check fire after every block (13 / 20 Ritz calls instead of 3); SSA_CHECK_RATIO=100
# keeps the check schedule of the uninstrumented run (same products, 3 Ritz calls)
for c in c2 c3; do
SSA_CHECK_RATIO=100 python scripts/prof_decompose.py $c > gpurun_out/pd_$c.log 2>&1 && SSA_CHECK_RATIO=100 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_dec_$c.csv python scripts/prof_decompose.py $c > /dev/null 2>&1; echo "$c $?"; cat gpurun_out/pd_$c.log; python scripts/launch_summary.py gpurun_out/launches_dec_$c.csv | head -16
done
