out=gpurun_out/b03; mkdir -p $out
timeout 300 python scripts/bench_tall_c5.py 2>&1 | tail -12
bash scripts/gpu_bench.sh b03 c3 c2 c4
timeout 1200 python -m pytest tests -m gpu -q -x --timeout 900 > $out/pytest.log 2>&1; tail -3 $out/pytest.log
