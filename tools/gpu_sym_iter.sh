# FAST-SYM kernel iteration: parity tests, old vs new vs variants timing, ncu of the default build
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout -s KILL 300 python -m pytest tests/test_fast_sym.py -m gpu -q -x -p no:cacheprovider > gpurun_out/t_sym.log 2>&1; echo "tests rc=$?" >> gpurun_out/t_sym.log
timeout -s KILL 300 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "fast_sym or sym" >> gpurun_out/t_sym.log 2>&1; echo "tests2 rc=$?" >> gpurun_out/t_sym.log
for i in 1 2; do
for v in ${VARIANTS:-old}; do echo "== $v" >> gpurun_out/time.log; BD_LIB_PATH=paper_1703_02484_b200/_lib/variants/libbd_$v.so timeout -s KILL 120 python tools/time_force.py 131072:fast-sym 65536:fast-sym >> gpurun_out/time.log 2>&1; done
echo "== new" >> gpurun_out/time.log
timeout -s KILL 120 python tools/time_force.py 131072:fast-sym 65536:fast-sym >> gpurun_out/time.log 2>&1
done
if [ "${NCU:-1}" = 1 ]; then
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:k_allpairs_sym -s 1 -c 1 -o gpurun_out/prof_sym_new python tools/prof_force.py 131072 fast-sym 2 > gpurun_out/ncu_new.log 2>&1
fi
tail -4 gpurun_out/t_sym.log; cat gpurun_out/time.log
