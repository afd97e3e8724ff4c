SSA_GRAM_TRACE=1 python scripts/bench_tall1.py 3 201601 32 32 2>&1 | tail -16
SSA_GRAM_TRACE=1 python scripts/bench_tall1.py 0 201601 224 32 2>&1 | tail -16
