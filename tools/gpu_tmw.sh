# TMEM warp tier: warp-tier parity tests, then A/B vs the register warp tier (DABS_TMW=0)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "batch_parity or generation_parity or sampled" > gpurun_out/pytest_tmw.log 2>&1; echo "pytest rc $?"; tail -15 gpurun_out/pytest_tmw.log
for w in ${WORKLOADS:-K2000s TSP32 GS800}; do
  for v in 0 1; do
    DABS_TMW=$v timeout 600 python bench.py --workload $w --no-cpu-baseline --no-e2e --no-tts --no-async --no-jump > gpurun_out/tmw_${w}_$v.log 2>&1; echo "bench $w TMW=$v rc $?"
    python - "$w" "$v" <<'PY'
import json, sys
w, v = sys.argv[1], sys.argv[2]
d = json.loads(open(f"gpurun_out/tmw_{w}_{v}.log").read().strip().split("\n")[-1])
print(w, "TMW=" + v, "%.4g" % d["value"], round(d["roofline"]["frac"], 3), d["config"]["slots_per_gpu"], "%.1f ms" % d["ms_per_step"], {k: round(x["frac"], 3) for k, x in d.get("per_rule", {}).items()})
PY
  done
done
