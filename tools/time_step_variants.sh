# maintenance-kernel timing per library variant: cfg3 phases + cfg2/cfg4 short runs
cd $GRAFT_REPO_ROOT
for f in paper_1703_02484_b200/_lib/libbd_b200.so paper_1703_02484_b200/_lib/variants/*.so; do
  echo "== $f"
  BD_LIB_PATH=$f python tools/phase_probe.py 131072 fast-sym 2>&1 | head -2
  BD_LIB_PATH=$f python tools/run_configs.py --cfg 2 4 --steps 10 --no-cpu 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    r=json.loads(l); print(r['config'], 'ms/step', round(r['ms_per_step'],3), 'maintain', round(r['phase_ms']['maintain'],3), 'GB/s', round(r['maintain_roofline']['achieved']), 'valid', r['valid_every_checked_step'])"
done
