# round-2 GPU check: parity suites, A/B at config sizes, reference suite, sanitizers, bench
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
nproc > gpurun_out/nproc.txt
T() { local name=$1; shift; local t0=$(date +%s); timeout -s KILL ${TLIM:-1500} "$@" > gpurun_out/$name.log 2>&1; echo "$name rc=$? $(( $(date +%s) - t0 ))s" >> gpurun_out/summary.txt; }
for s in ${SUITES:-gpu ab ref san bench}; do
  case $s in
    gpu) T pytest_gpu python -m pytest tests -m gpu -q -x --deselect tests/test_ab_configs.py --deselect tests/test_reference_suite_gpu.py --deselect tests/test_sanitizer_gpu.py -p no:cacheprovider ;;
    ab) T pytest_ab python -m pytest tests/test_ab_configs.py -m gpu -q -s -p no:cacheprovider ;;
    ref) T pytest_ref python -m pytest tests/test_reference_suite_gpu.py -m gpu -q -s -p no:cacheprovider ;;
    san) T pytest_san python -m pytest tests/test_sanitizer_gpu.py -m gpu -q -p no:cacheprovider ;;
    bench) T bench python bench.py ${BENCH_ARGS:-} ;;
    benchref) T bench_ref python bench.py --impl reference --steps 3 --warmup 1 ;;
    smoke) T smoke python -c "import __graft_entry__ as g; g.smoke()" ;;
  esac
done
cat gpurun_out/summary.txt
for f in gpurun_out/*.log; do echo "== $f"; tail -n 4 $f | cut -c1-600; done
