#!/bin/bash
# ncu --set full of the register-FFT passes of one X·V and one Xᵀ·U block product (c5 by default).
# Usage: bash scripts/gpu_prof_rpass.sh <tag> [config]
tag=${1:-prof}; cfg=${2:-c5}; out=gpurun_out/$tag; mkdir -p $out
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1 || { tail -20 $out/build.log; exit 1; }
timeout 300 python scripts/prof_products.py $cfg fft 64 2 || exit 1
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:rpass_ --launch-skip 7 --launch-count 6 \
  -o $out/rpass_$cfg python scripts/prof_products.py $cfg fft 64 1 > $out/ncu.log 2>&1
tail -3 $out/ncu.log
