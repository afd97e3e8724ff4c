#!/bin/bash
out=gpurun_out/s6; mkdir -p $out
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1 || { tail -20 $out/build.log; exit 1; }
timeout 300 python scripts/prof_products.py c5 fft 2>&1 | tail -2
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file $out/launches_c3.csv \
  python bench.py --config c3 --steps 2 --warmup 3 --no-cpu-baseline > $out/ncu_c3.log 2>&1
python scripts/launch_summary.py $out/launches_c3.csv > $out/launches_c3.summary.txt 2>&1; head -25 $out/launches_c3.summary.txt
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 > $out/pytest_gpu.log 2>&1
tail -3 $out/pytest_gpu.log
