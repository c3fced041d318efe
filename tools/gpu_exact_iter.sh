# EXACT kernel iteration: fast-path arithmetic check, EXACT parity tests, variant timing
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
L=gpurun_out/exact_iter.log
timeout -s KILL 600 python -m pytest tests/test_exact_fastpath_gpu.py -m gpu -q -x -p no:cacheprovider > $L 2>&1; echo "fastpath rc=$?" >> $L
timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py tests/test_ab_configs.py -m gpu -q -x -p no:cacheprovider >> $L 2>&1; echo "parity rc=$?" >> $L
for v in ${VARIANTS:-} new; do
  if [ "$v" = new ]; then LP=""; else LP=paper_1703_02484_b200/_lib/variants/libbd_$v.so; fi
  echo "== $v" >> $L
  BD_LIB_PATH=$LP timeout -s KILL 300 python tools/time_force.py 131072:exact 65536:exact 16384:exact >> $L 2>&1
done
tail -40 $L
if [ "${NCU:-0}" = 1 ]; then
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:k_allpairs -s 1 -c 1 -o gpurun_out/prof_exact python tools/prof_force.py 65536 exact 2 > gpurun_out/ncu_exact.log 2>&1
fi
