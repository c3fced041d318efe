# step-kernel change check: parity goldens on every driver + timings at the config sizes
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout -s KILL 400 python -m pytest tests/test_gpu_parity.py tests/test_ops.py tests/test_abp.py tests/test_msd.py -m gpu -q -x -p no:cacheprovider > gpurun_out/step_tests.log 2>&1; echo "rc=$?" >> gpurun_out/step_tests.log
BD_BLOCK_MAX_N=0 timeout -s KILL 300 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "bitwise or batched" > gpurun_out/step_tests_grid.log 2>&1; echo "rc=$?" >> gpurun_out/step_tests_grid.log
TAG=new timeout -s KILL 300 python tools/time_step.py ${CFGS:-cfg1 n4096 cfg2 cfg5 cfg3} > gpurun_out/steps.log 2>&1
tail -n 2 gpurun_out/step_tests.log; tail -n 2 gpurun_out/step_tests_grid.log; cat gpurun_out/steps.log
