# GPU check: build, parity tests (single-CTA and grid drivers), bench, multi-rank path
cd $GRAFT_REPO_ROOT
python -m paper_1703_02484_b200.build --force > gpurun_out/build.log 2>&1
make -s -C oracle >> gpurun_out/build.log 2>&1
timeout -s KILL 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
BD_BLOCK_MAX_N=0 timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "bitwise or batched or pair_list or sharded" > gpurun_out/pytest_gpu_grid.log 2>&1
timeout -s KILL 900 python bench.py ${BENCH_ARGS:-} > gpurun_out/bench.log 2>&1
if [ "$EXACT" = 1 ]; then
timeout -s KILL 900 python bench.py --steps 5 --warmup 3 --precision exact --no-cpu-baseline --no-e2e > gpurun_out/bench_exact.log 2>&1
fi
if [ "$MULTI" = 1 ]; then
BD_BENCH_GLOO=1 timeout -s KILL 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_multi.log 2>&1
fi
if [ "$REF" = 1 ]; then
timeout -s KILL 900 python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/bench_ref.log 2>&1
fi
for f in pytest_gpu pytest_gpu_grid bench bench_exact bench_multi bench_ref; do [ -f gpurun_out/$f.log ] && { echo "== $f"; tail -n 3 gpurun_out/$f.log | cut -c1-1500; }; done
