for c in c2 c3; do SSA_DEBUG=1 python scripts/debug_decompose.py $c auto > gpurun_out/dbg_$c.log 2>&1; echo "$c $?"; grep -E "ritz_svd|host ms" gpurun_out/dbg_$c.log | tail -8; done
