# A/B: warp tier vs two-warp CTA tier (DABS_W2=1) for n <= 2048 workloads (generation schedule)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
for w in ${WORKLOADS:-K2000s TSP32 GS800}; do
  for v in 0 1; do
    DABS_W2=$v timeout 600 python bench.py --workload $w --no-cpu-baseline --no-e2e --no-tts --no-async --no-jump > gpurun_out/ab_${w}_$v.log 2>&1; echo "bench $w W2=$v rc $?"
    python - "$w" "$v" <<'PY'
import json, sys
w, v = sys.argv[1], sys.argv[2]
d = json.loads(open(f"gpurun_out/ab_{w}_{v}.log").read().strip().split("\n")[-1])
print(w, "W2=" + v, "%.4g" % d["value"], d["roofline"]["bound"], round(d["roofline"]["frac"], 3), d["config"].get("threads_per_search"), {k: round(x["frac"], 3) for k, x in d.get("per_rule", {}).items()})
PY
  done
done
