mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
for w in K2000s TSP32; do
  DABS_TMW=1 timeout 600 python bench.py --workload $w --no-cpu-baseline --no-e2e --no-tts --no-async --no-jump > gpurun_out/tmw2_${w}.log 2>&1; echo "bench $w rc $?"
  python - "$w" <<'PY'
import json, sys
w = sys.argv[1]
d = json.loads(open(f"gpurun_out/tmw2_{w}.log").read().strip().split("\n")[-1])
print(w, "TMW=1 occ8", "%.4g" % d["value"], round(d["roofline"]["frac"], 3), d["config"]["slots_per_gpu"], "%.1f ms" % d["ms_per_step"], {k: round(x["frac"], 3) for k, x in d.get("per_rule", {}).items()})
PY
done
