mkdir -p gpurun_out/dump
for c in c2 c3 c4; do SSA_DEBUG=1 SSA_DUMP_T=gpurun_out/dump/$c python scripts/debug_decompose.py $c auto > gpurun_out/dbg_$c.log 2>&1; echo "$c $?"; grep -E "ritz_svd|host ms" gpurun_out/dbg_$c.log | tail -8; done
timeout 120 python scripts/bench_jacobi.py 2>&1 | tail -8
