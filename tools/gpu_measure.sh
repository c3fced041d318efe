# round measurement set (outputs in gpurun_out/; summaries are copied into profiles/ by hand)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
S=${WHAT:-"prof bench configs long"}
for w in $S; do case $w in
  prof) PROFILES=${PROFILES:-"sym exact step launches"} bash tools/profile.sh > gpurun_out/profile.log 2>&1 ;;
  bench) timeout -s KILL 900 python bench.py > gpurun_out/bench_m.log 2>gpurun_out/bench_m.err ;;
  benchexact) timeout -s KILL 900 python bench.py --steps 10 --warmup 3 --precision exact --no-cpu-baseline > gpurun_out/bench_exact.log 2>&1 ;;
  benchref) timeout -s KILL 1500 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.log 2>&1 ;;
  configs) timeout -s KILL 1500 python tools/run_configs.py --cfg 1 2 5 4 > gpurun_out/configs.jsonl 2>gpurun_out/configs.err ;;
  long) timeout -s KILL 900 python tools/run_configs.py --cfg 3 --no-cpu > gpurun_out/cfg3_long.jsonl 2>gpurun_out/cfg3_long.err ;;
esac; echo "$w done rc=$?" >> gpurun_out/measure.txt; done
cat gpurun_out/measure.txt; ls -la gpurun_out
