# quick GPU check of selected test files (+ force timing)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout -s KILL ${TLIM:-900} python -m pytest ${TESTS:-tests/test_fast_sym.py} -m gpu -q -x -p no:cacheprovider > gpurun_out/quick.log 2>&1; echo "rc=$?" >> gpurun_out/quick.log
[ -n "$TIME" ] && timeout -s KILL 120 python tools/time_force.py 131072:fast-sym 65536:fast-sym 16384:fast-sym >> gpurun_out/quick.log 2>&1
tail -25 gpurun_out/quick.log
