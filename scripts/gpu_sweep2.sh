python scripts/sweep_k.py c2 16 3,4
python scripts/sweep_k.py c1 8 3,4,6
python scripts/sweep_k.py c4 16,32 2,3,4
python scripts/sweep_k.py c3 32 3,4,5
SSA_FIRST_BLOCKS=99 python scripts/sweep_k.py c4 16 3
