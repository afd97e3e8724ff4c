timeout 900 python -m pytest tests/ -m gpu -x -q -k "decompose or edge or reconstruct or band or c3_noiseless" > gpurun_out/pytest_q.log 2>&1; echo "pytest $?"; tail -3 gpurun_out/pytest_q.log
timeout 900 python scripts/sweep_warm.py c1,c2,c3,c4,c5 d d
echo LEGACY; SSA_ORTH_LEGACY=1 timeout 900 python scripts/sweep_warm.py c2,c3 d d
for c in c2 c3; do SSA_DEBUG=1 python scripts/debug_decompose.py $c auto 2>&1 | grep "host ms"; done
