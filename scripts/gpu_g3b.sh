timeout 900 python -m pytest tests/ -m gpu -x -q -k "tall or decompose or edge or c3_noiseless or orth" > gpurun_out/pytest_q.log 2>&1; echo "pytest $?"; tail -3 gpurun_out/pytest_q.log
for v in 1 3; do for c in c3 c4 c5; do echo "V=$v $c: $(SSA_GRAM_V=$v python scripts/prof_decompose.py $c 2>&1 | tail -1)"; done; done
