# GPU check: build, parity tests (single-CTA and grid drivers), bench, launch list
cd $GRAFT_REPO_ROOT
python -m paper_1703_02484_b200.build --force > gpurun_out/build.log 2>&1
make -s -C oracle >> gpurun_out/build.log 2>&1
timeout -s KILL 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
BD_BLOCK_MAX_N=0 timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "bitwise or batched or pair_list" > gpurun_out/pytest_gpu_grid.log 2>&1
timeout -s KILL 900 python bench.py --steps 20 --warmup 3 > gpurun_out/bench.log 2>&1
timeout -s KILL 900 python bench.py --steps 5 --warmup 3 --precision exact --no-cpu-baseline --no-e2e > gpurun_out/bench_exact.log 2>&1
if [ "$NCU" = 1 ]; then
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_bench.log 2>&1
fi
for f in pytest_gpu pytest_gpu_grid bench bench_exact; do echo "== $f"; tail -n 4 gpurun_out/$f.log; done
