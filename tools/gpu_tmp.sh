cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
L=gpurun_out/steps.log; rm -f $L
CF=${CFGS:-"n4096 n8192 cfg2 cfg5 cfg3"}
for i in 1 2; do
TAG=default timeout -s KILL 600 python tools/time_step.py $CF >> $L 2>&1
TAG=big0 BD_BIG_MIN_N=0 timeout -s KILL 600 python tools/time_step.py $CF >> $L 2>&1
done
