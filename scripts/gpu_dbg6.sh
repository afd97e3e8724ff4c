for c in c4 c3 c5; do SSA_DEBUG=1 timeout 300 python scripts/debug_decompose.py $c auto > gpurun_out/dbg_$c.log 2>&1; echo "$c $?"; grep -E "\] ritz |host ms" gpurun_out/dbg_$c.log | tail -12; done
