timeout 900 python scripts/sweep_warm.py c2,c3 d d
echo ORTH2; SSA_ORTH2=1 timeout 900 python scripts/sweep_warm.py c2,c3 d d
echo FAST; SSA_ORTH_FAST=1 timeout 900 python scripts/sweep_warm.py c2,c3 d d
echo NOFIRST; SSA_FIRST_BLOCKS=100 timeout 900 python scripts/sweep_warm.py c2,c3 d d
