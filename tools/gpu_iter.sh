# iteration check of a kernel change: build, parity tests, per-flip timing (DABS_TIMING variant), quick bench lines
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 1500 python -m pytest ${TESTS:-tests/test_gpu_parity.py tests/test_gpu_parity_nt512.py} -m gpu -x -q > gpurun_out/pytest_iter.log 2>&1; echo "pytest rc $?"; tail -5 gpurun_out/pytest_iter.log
if [ -n "$TIMING_LIB" ]; then
  DABS_LIB=$TIMING_LIB timeout 900 python tools/timing.py ${CFG:-R32K} 2 ${MASKS:-1,2,4,8,16,31} > gpurun_out/timing_iter.txt 2>&1; echo "timing rc $?"; cat gpurun_out/timing_iter.txt
fi
for w in ${WORKLOADS:-R32K K2000s}; do
  timeout 600 python bench.py --workload $w --no-cpu-baseline --no-e2e --no-tts --no-async --no-jump > gpurun_out/q_$w.log 2>&1; echo "bench $w rc $?"
  python - "$w" <<'PY'
import json, sys
w = sys.argv[1]
d = json.loads(open(f"gpurun_out/q_{w}.log").read().strip().split("\n")[-1])
print(w, "%.4g" % d["value"], d["roofline"]["bound"], round(d["roofline"]["frac"], 3), {k: round(v["frac"], 3) for k, v in d.get("per_rule", {}).items()})
PY
done
