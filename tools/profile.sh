# ncu evidence for profiles/ (run under gpurun; one GPU; never multi-rank).
# PROFILES selects the captures (default: all); keep the outputs < 64 MiB per call.
cd $GRAFT_REPO_ROOT
python -m paper_1703_02484_b200.build > /dev/null 2>&1
mkdir -p gpurun_out
P=${PROFILES:-"launches fast sym exact step"}
for what in $P; do
  case $what in
    launches)  # launch list of a short bench (cold-cache, serialised: compare shares)
      timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
        python bench.py --steps 3 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch_bench.log 2>&1 ;;
    fast)      # FAST all-pairs kernel (N = 131,072)
      timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:k_allpairs_fast -s 1 -c 1 \
        -o gpurun_out/prof_allpairs_fast python tools/prof_force.py 131072 fast 2 > gpurun_out/ncu_ap.log 2>&1 ;;
    sym)       # FAST-SYM pair kernel (N = 131,072; the bench default)
      timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:k_allpairs_sym -s 1 -c 1 \
        --metrics sm__sass_thread_inst_executed_op_dfma_pred_on.sum,sm__sass_thread_inst_executed_op_dmul_pred_on.sum,sm__sass_thread_inst_executed_op_dadd_pred_on.sum \
        -o gpurun_out/prof_allpairs_sym python tools/prof_force.py 131072 fast-sym 2 > gpurun_out/ncu_aps.log 2>&1 ;;
    exact)     # EXACT all-pairs kernel (N = 131,072)
      timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k k_allpairs -c 1 \
        --metrics sm__sass_thread_inst_executed_op_dfma_pred_on.sum,sm__sass_thread_inst_executed_op_dmul_pred_on.sum,sm__sass_thread_inst_executed_op_dadd_pred_on.sum \
        -o gpurun_out/prof_allpairs_exact python tools/prof_force.py 131072 exact 1 > gpurun_out/ncu_apx.log 2>&1 ;;
    step)      # persistent step kernel (cfg3 state after warm-up)
      timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:k_step_tri_grid -s 2 -c 1 \
        -o gpurun_out/prof_step_tri python bench.py --steps 1 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/ncu_step.log 2>&1 ;;
  esac
done
ls -la gpurun_out
