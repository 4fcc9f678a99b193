mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for wv in ${WAVES:-4 8}; do
DABS_WAVES=$wv timeout 900 python bench.py --workload ${W:-R32K} --no-cpu-baseline --no-e2e --no-tts --no-async --no-jump > gpurun_out/waves_$wv.log 2>&1; echo "rc $?"
python - $wv <<'PY'
import json, sys
d = json.loads(open(f"gpurun_out/waves_{sys.argv[1]}.log").read().strip().split("\n")[-1])
print("waves", sys.argv[1], "%.4g" % d["value"], round(d["roofline"]["frac"], 3), d["config"]["slots_per_gpu"], d["ms_per_step"], {k: round(x["frac"], 3) for k, x in d.get("per_rule", {}).items()})
PY
done
