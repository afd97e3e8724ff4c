python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 300 python scripts/bench_tall_c5.py
SSA_GRAM_TC=0 timeout 300 python scripts/bench_tall_c5.py 2>&1 | head -3
