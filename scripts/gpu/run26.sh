python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
mkdir -p gpurun_out/r26
SSA_GRAM_SELF=3 timeout 600 ncu --set full --import-source on --clock-control none -k regex:"gram_self" -s 1 -c 1 -o gpurun_out/r26/self python scripts/prof_tall.py 3 64 64 > gpurun_out/r26/ncu_self.log 2>&1
tail -1 gpurun_out/r26/ncu_self.log
