python scripts/time_plan.py c2 c3 c4 c5
SSA_PLAN_CORR=1 python scripts/time_plan.py c4
timeout 900 python -m pytest tests/ -m gpu -x -q -k "shaped or c4 or mask or edge or band or weights or wcor" > gpurun_out/pytest_q.log 2>&1; echo "pytest $?"; tail -2 gpurun_out/pytest_q.log
