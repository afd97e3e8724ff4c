python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 600 python -m pytest tests/test_gpu_tall.py -q -x 2>&1 | tail -3
timeout 300 python scripts/bench_tall_c5.py
SSA_GRAM_SELF=0 timeout 300 python scripts/bench_tall_c5.py | head -1
