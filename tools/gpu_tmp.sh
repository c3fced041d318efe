cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
L=gpurun_out/steps.log; rm -f $L
CF=${CFGS:-"cfg1 n4096 cfg2 cfg5 cfg3"}
for v in ${VARIANTS:-} new; do
  if [ "$v" = new ]; then LP=""; else LP=paper_1703_02484_b200/_lib/variants/libbd_$v.so; fi
  TAG=$v BD_LIB_PATH=$LP timeout -s KILL 600 python tools/time_step.py $CF >> $L 2>&1
done
cat $L
