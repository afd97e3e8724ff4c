python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
mkdir -p gpurun_out/r20
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"gram_self" -s 1 -c 1 -o gpurun_out/r20/self python scripts/prof_tall.py 3 64 64 > gpurun_out/r20/ncu_self.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"update_tc2" -s 1 -c 1 -o gpurun_out/r20/upd python scripts/prof_tall.py 1 128 64 > gpurun_out/r20/ncu_upd.log 2>&1
tail -2 gpurun_out/r20/ncu_self.log
