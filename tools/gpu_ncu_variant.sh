# ncu --set full of the FAST-SYM pair kernel of one variant build (VARIANT=name or "new")
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for v in ${VARIANTS:-new}; do
  if [ "$v" = new ]; then LP=""; else LP=paper_1703_02484_b200/_lib/variants/libbd_$v.so; fi
  BD_LIB_PATH=$LP timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:k_allpairs_sym -s 1 -c 1 -o gpurun_out/prof_sym_$v python tools/prof_force.py 131072 fast-sym 2 > gpurun_out/ncu_$v.log 2>&1
done
ls -la gpurun_out
