SSA_ORTH_FAST=1 python scripts/debug_decompose.py c2 auto > gpurun_out/plain_dbg3.log 2>&1 && SSA_ORTH_FAST=1 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_orthfast.csv python scripts/debug_decompose.py c2 auto > /dev/null 2>&1
python scripts/launch_summary.py gpurun_out/launches_orthfast.csv | head -20
python scripts/debug_decompose.py c2 auto > gpurun_out/plain_dbg3.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_legacy.csv python scripts/debug_decompose.py c2 auto > /dev/null 2>&1
python scripts/launch_summary.py gpurun_out/launches_legacy.csv | head -20
