# time the FAST all-pairs kernel of every built variant (tools/build_variants.py) at N = 131,072
cd $GRAFT_REPO_ROOT
echo "== in-tree"; python tools/time_force.py ${SPECS:-131072:fast 131072:fast}
for f in paper_1703_02484_b200/_lib/variants/*.so; do
  echo "== $f"; BD_LIB_PATH=$f python tools/time_force.py ${SPECS:-131072:fast 131072:fast} | tail -${TAILN:-20}
done
