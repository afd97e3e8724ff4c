python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 400 python scripts/sweep_k.py c2 16,24,32 3,4,6
timeout 400 python scripts/sweep_k.py c3 16,32 4,6
timeout 400 python scripts/sweep_k.py c4 16,32 4,6
