python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
mkdir -p gpurun_out/r12
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r12/smoke.log 2>&1; tail -2 gpurun_out/r12/smoke.log
timeout 900 python bench.py > gpurun_out/r12/bench_c5.json 2> gpurun_out/r12/bench_c5.err
tail -c 400 gpurun_out/r12/bench_c5.json
timeout 1800 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/r12/pytest_gpu.log 2>&1
tail -5 gpurun_out/r12/pytest_gpu.log
torchrun --standalone --nnodes 1 --nproc-per-node 1 bench.py --gpus 1 --shard --steps 2 --warmup 1 --config c3 > gpurun_out/r12/shard_c3.json 2> gpurun_out/r12/shard_c3.err
tail -c 400 gpurun_out/r12/shard_c3.json
