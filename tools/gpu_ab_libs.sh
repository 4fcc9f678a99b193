# A/B of library builds (DABS_LIB) on quick bench lines: LIBS="a.so b.so" WORKLOADS="..."
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
for w in ${WORKLOADS:-K2000s TSP32 GS800}; do
  for lib in default ${LIBS}; do
    tag=$(basename $lib .so)
    if [ "$lib" = default ]; then unset DABS_LIB; else export DABS_LIB=$lib; fi
    timeout 600 python bench.py --workload $w --no-cpu-baseline --no-e2e --no-tts --no-async --no-jump ${EXTRA} > gpurun_out/ab_${w}_$tag.log 2>&1; echo "bench $w $tag rc $?"
    python - "$w" "$tag" <<'PY'
import json, sys
w, v = sys.argv[1], sys.argv[2]
d = json.loads(open(f"gpurun_out/ab_{w}_{v}.log").read().strip().split("\n")[-1])
print(w, v, "%.4g" % d["value"], d["roofline"]["bound"], round(d["roofline"]["frac"], 3), {k: round(x["frac"], 3) for k, x in d.get("per_rule", {}).items()})
PY
  done
done
unset DABS_LIB
