timeout 900 python -m pytest tests/ -m gpu -x -q -k "c5 or decompose or edge" > gpurun_out/pytest_q.log 2>&1; echo "pytest $?"; tail -2 gpurun_out/pytest_q.log
timeout 900 python scripts/sweep_warm.py c5 d d
SSA_NO_NEAR_CHECK=1 python scripts/prof_decompose.py c5 > /dev/null 2>&1 && SSA_NO_NEAR_CHECK=1 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_dec_c5.csv python scripts/prof_decompose.py c5 > /dev/null 2>&1; python scripts/launch_summary.py gpurun_out/launches_dec_c5.csv | head -16
