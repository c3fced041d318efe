# O(N) step driver variants at the config sizes (tools/time_step.py)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
CF=${CFGS:-"cfg1 n4096 cfg2"}
TAG=default timeout -s KILL 600 python tools/time_step.py $CF >> gpurun_out/steps.log 2>&1
TAG=cluster16 BD_CLUSTER_MAX_N=70000 BD_CLUSTER_SIZE=16 timeout -s KILL 600 python tools/time_step.py $CF >> gpurun_out/steps.log 2>&1
TAG=cluster8 BD_CLUSTER_MAX_N=70000 BD_CLUSTER_SIZE=8 timeout -s KILL 600 python tools/time_step.py $CF >> gpurun_out/steps.log 2>&1
TAG=grid BD_BLOCK_MAX_N=0 timeout -s KILL 600 python tools/time_step.py $CF >> gpurun_out/steps.log 2>&1
cat gpurun_out/steps.log
