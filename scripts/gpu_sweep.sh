python scripts/sweep_k.py c2 16,24,32,48 3,4,6
python scripts/sweep_k.py c3 16,32,48 2,3,4
python scripts/sweep_k.py c1 8,16,32 3,4,6
