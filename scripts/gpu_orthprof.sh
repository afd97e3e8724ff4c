SSA_ORTH_FAST=1 python scripts/debug_decompose.py c2 auto > gpurun_out/plain_op.log 2>&1 && SSA_ORTH_FAST=1 ncu --set full --clock-control none --import-source on -k regex:"orth_solve|apply_inplace" -s 10 -c 4 -o gpurun_out/prof_orth python scripts/debug_decompose.py c2 auto > gpurun_out/ncu_orth.log 2>&1
echo "ncu $?"
