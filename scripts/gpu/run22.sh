python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
SSA_GRAM_SELF=2 timeout 300 python scripts/bench_tall_c5.py 2>&1 | head -1
mkdir -p gpurun_out/r22
SSA_GRAM_SELF=2 timeout 600 ncu --set full --import-source on --clock-control none -k regex:"gram_self" -s 1 -c 1 -o gpurun_out/r22/self4 python scripts/prof_tall.py 3 64 64 > gpurun_out/r22/ncu_self.log 2>&1
