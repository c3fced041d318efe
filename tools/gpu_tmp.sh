cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
L=gpurun_out/exact2.log
timeout -s KILL 900 python -m pytest tests/test_exact_fastpath_gpu.py tests/test_gpu_parity.py tests/test_ab_configs.py tests/test_msd.py -m gpu -q -x -p no:cacheprovider > $L 2>&1; echo "rc=$?" >> $L
timeout -s KILL 300 python tools/time_force.py 131072:exact 65536:exact 16384:exact 8192:exact 4096:exact 1024:exact >> $L 2>&1
tail -12 $L
