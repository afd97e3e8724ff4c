timeout 900 python scripts/sweep_warm.py c1,c2,c3,c4 d d
echo BLOCKING; SSA_BLOCKING_SYNC=1 timeout 900 python scripts/sweep_warm.py c1,c2,c3,c4 d d
