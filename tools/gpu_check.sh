set -x
cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
python -m paper_1703_02484_b200.build --force > gpurun_out/build.log 2>&1
make -s -C oracle >> gpurun_out/build.log 2>&1
timeout -s KILL 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
BD_BLOCK_MAX_N=0 timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "bitwise or batched" > gpurun_out/pytest_gpu_grid.log 2>&1
timeout -s KILL 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.log 2>&1
tail -5 gpurun_out/pytest_gpu.log gpurun_out/pytest_gpu_grid.log gpurun_out/bench.log
