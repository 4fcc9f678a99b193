mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
DABS_DEBUG_OCC=1 timeout 900 python bench.py --no-cpu-baseline --no-e2e --no-tts --no-async --no-jump > gpurun_out/occ_r32k.log 2>&1; echo "rc $?"; grep "dabs: occ" gpurun_out/occ_r32k.log | head -3
python - <<'PY'
import json
d = json.loads(open("gpurun_out/occ_r32k.log").read().strip().split("\n")[-1])
print("R32K", "%.4g" % d["value"], round(d["roofline"]["frac"], 3), d["config"]["slots_per_gpu"], {k: round(x["frac"], 3) for k, x in d.get("per_rule", {}).items()})
PY
