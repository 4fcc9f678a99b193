# warp tier A/B: sigma table (DABS_WARP_LUT builds) and waves per generation
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
run() {  # tag, env...
  tag=$1; shift
  env "$@" timeout 600 python bench.py --workload $w --no-cpu-baseline --no-e2e --no-tts --no-async --no-jump > gpurun_out/abw_${w}_$tag.log 2>&1
  python - "$w" "$tag" <<'PY'
import json, sys
w, v = sys.argv[1], sys.argv[2]
d = json.loads(open(f"gpurun_out/abw_{w}_{v}.log").read().strip().split("\n")[-1])
print(w, v, "%.4g" % d["value"], round(d["roofline"]["frac"], 3), d["config"]["slots_per_gpu"], "%.1f ms/step" % d["ms_per_step"], {k: round(x["frac"], 3) for k, x in d.get("per_rule", {}).items()})
PY
}
for w in ${WORKLOADS:-K2000s TSP32 GS800}; do
  run base
  run wlut DABS_LIB=ab/libdabs_wlut.so
  run wlut20 DABS_LIB=ab/libdabs_wlut20.so
  run waves8 DABS_WAVES=8
  run waves16 DABS_WAVES=16
done
