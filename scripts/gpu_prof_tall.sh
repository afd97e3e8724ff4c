#!/bin/bash
# ncu --set full of the solver's tall-skinny kernels at c5's K-side size (one launch each), plus live
# timings (scripts/bench_tall_c5.py).  Usage: bash scripts/gpu_prof_tall.sh <tag>
tag=${1:-tall}; out=gpurun_out/$tag; mkdir -p $out
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1 || { tail -20 $out/build.log; exit 1; }
timeout 300 python scripts/bench_tall_c5.py > $out/bench_tall_c5.txt 2>&1; cat $out/bench_tall_c5.txt
for spec in "3 64 64 gram_self" "5 128 64 gram_tc3" "1 128 64 update_tc2"; do
  set -- $spec
  timeout 600 ncu --set full --clock-control none -k regex:$4 --launch-skip 1 --launch-count 1 -o $out/prof_${4}_$2 \
    python scripts/prof_tall.py $1 $2 $3 > $out/ncu_$4.log 2>&1
done
for f in $out/prof_*.ncu-rep; do python scripts/ncu_brief.py $f; done > $out/prof_tall_c5.summary.txt 2>&1
cat $out/prof_tall_c5.summary.txt
