cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
L=gpurun_out/phase.log
for n in 131072 16384 1024; do echo "== $n" >> $L; timeout -s KILL 300 python tools/phase_probe.py $n fast-sym >> $L 2>&1; done
cat $L
