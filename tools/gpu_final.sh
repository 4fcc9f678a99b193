# round-2 final check: all -m gpu tests, smoke, the default bench line (R32K) and full lines of the other workloads
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 1800 python -m pytest tests -m gpu -x -q --durations=8 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?"; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc $?"; tail -1 gpurun_out/smoke.log
timeout 1200 python bench.py > gpurun_out/final_R32K.log 2>&1; echo "bench R32K rc $?"
for w in ${WORKLOADS:-K2000s TSP32 GS800}; do
  timeout 900 python bench.py --workload $w > gpurun_out/final_$w.log 2>&1; echo "bench $w rc $?"
done
for w in R32K ${WORKLOADS:-K2000s TSP32 GS800}; do
python - $w <<'PY'
import json, sys
w = sys.argv[1]
d = json.loads(open(f"gpurun_out/final_{w}.log").read().strip().split("\n")[-1])
print(w, "%.4g" % d["value"], d["roofline"]["bound"], round(d["roofline"]["frac"], 3), "e2e %.4g" % d["e2e"]["value"], d["clocks"], {k: round(x["frac"], 3) for k, x in d.get("per_rule", {}).items()})
print("  tts", json.dumps(d.get("time_to_target"))[:300])
print("  cpu", json.dumps(d.get("cpu_baseline"))[:300])
PY
done
