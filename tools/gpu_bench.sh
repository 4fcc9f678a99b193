# GPU bench pass: record the R32K target, bench lines, launch list + one ncu full capture
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
cp profiles/targets.json gpurun_out/targets.json
if [ -n "$RECORD" ]; then
  timeout 400 python tools/record_target.py --workload R32K --seconds 60 --seeds 2 --out gpurun_out/targets.json > gpurun_out/record_r32k.log 2>&1
  python - <<'PY'
import json; d=json.load(open("gpurun_out/targets.json")); d["R32K"].update(limit_s=30, runs=2); json.dump(d, open("gpurun_out/targets.json","w"), indent=1)
PY
  cp gpurun_out/targets.json profiles/targets.json
fi
for w in ${WORKLOADS:-R32K K2000s TSP32 GS800}; do
  timeout 900 python bench.py --workload $w > gpurun_out/bench_$w.log 2>&1; echo "bench $w rc $?"
  tail -1 gpurun_out/bench_$w.log | cut -c1-400
done
